"""One-off probe of the GPU box: host CPU, PCIe pinned H2D/D2H bandwidth, HBM copy."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
except Exception as e:
    out["lscpu"] = str(e)
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["smi"] = subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK,PCIE"], capture_output=True, text=True).stdout[-3000:]
dev = torch.device("cuda:0")
for nbytes in (256 << 20, 1208 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); h.copy_(d, non_blocking=True); e2.record()
    torch.cuda.synchronize()
    out[f"h2d_GBps_{nbytes>>20}MB"] = nbytes / e0.elapsed_time(e1) / 1e6
    out[f"d2h_GBps_{nbytes>>20}MB"] = nbytes / e1.elapsed_time(e2) / 1e6
    # bidirectional
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); out[f"bidir_GBps_{nbytes>>20}MB"] = 2 * nbytes / (time.perf_counter() - t) / 1e9
print(json.dumps(out, indent=1))
