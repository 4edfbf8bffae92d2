import torch, time
a = torch.rand(4096, 4096, dtype=torch.float64, device="cuda")
b = torch.rand(4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(2): c = a @ b
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): c = a @ b
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
print(f"DGEMM 4096^3: {2*4096**3/dt/1e12:.1f} TFLOP/s")
x = torch.rand(1 << 26, dtype=torch.float64, device="cuda")
y = torch.rand(1 << 26, dtype=torch.float64, device="cuda") + 1
for _ in range(2): z = x / y
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): z = x / y
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print(f"fp64 divide: {(1<<26)/dt/1e9:.1f} G div/s ({(1<<26)*24/dt/1e9:.0f} GB/s)")
