import os, sys, time, subprocess
import torch
dev = torch.device("cuda", 0)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("props pci:", bus)
out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", "0"], capture_output=True, text=True).stdout.strip()
print("nvidia-smi bus id:", out)
busid = out.lower()
# sysfs wants 0000:xx:yy.z (nvidia-smi prints 00000000:xx:yy.z)
if busid.count(":") == 2 and len(busid.split(":")[0]) == 8:
    busid = busid[4:]
p = f"/sys/bus/pci/devices/{busid}"
for f in ("local_cpulist", "numa_node"):
    try: print(f, open(os.path.join(p, f)).read().strip())
    except Exception as e: print(f, "n/a", e)
print("cpus:", os.cpu_count(), "affinity:", len(os.sched_getaffinity(0)))
try:
    print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500])
except Exception as e:
    print(e)
def h2d(tag):
    xh = torch.empty((131072, 16384), dtype=torch.float32, pin_memory=True)
    xh.fill_(1.0)
    xd = torch.empty((131072, 16384), device=dev)
    for k in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter(); xd.copy_(xh, non_blocking=True); torch.cuda.synchronize()
        print(f"{tag}: {xh.numel()*4/(time.perf_counter()-t0)/1e9:.1f} GB/s")
    del xh, xd; torch.cuda.empty_cache()
h2d("default affinity")
try:
    local = open(os.path.join(p, "local_cpulist")).read().strip()
    cpus = set()
    for part in local.split(","):
        a, _, b = part.partition("-"); cpus.update(range(int(a), int(b or a) + 1))
    allc = set(range(os.cpu_count()))
    os.sched_setaffinity(0, cpus); h2d(f"local cpus ({len(cpus)})")
    rem = allc - cpus
    if rem:
        os.sched_setaffinity(0, rem); h2d(f"remote cpus ({len(rem)})")
except Exception as e:
    print("affinity test failed:", e)
