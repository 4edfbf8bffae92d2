import sys, time
sys.path.insert(0, '.')
import torch, numpy as np
dev = torch.device("cuda", 0)
v = torch.rand((131072, 64), device=dev)
def t(fn, name):
    for k in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
        print(f"{name:40s} {1e3*(time.perf_counter()-t0):7.2f} ms")
    return out
t(lambda: v.detach().to("cpu", dtype=torch.float64).numpy(), "to(cpu, f64) [current]")
t(lambda: v.double().cpu().numpy(), "device double -> cpu pageable")
t(lambda: v.cpu().numpy().astype(np.float64), "cpu pageable -> astype")
def pinned():
    d = v.double()
    h = torch.empty(d.shape, dtype=torch.float64, pin_memory=True)
    h.copy_(d)
    return h.numpy()
t(pinned, "device double -> pinned")
def pinned32():
    h = torch.empty(v.shape, dtype=torch.float32, pin_memory=True)
    h.copy_(v)
    return h.numpy().astype(np.float64)
t(pinned32, "pinned f32 -> astype")
