"""Probe of the GPU box host for the config-5 end-to-end path: host RAM, time to pin the
config-5 K (77.3 GB) and values (32.7 GB) buffers, and large pinned H2D / D2H / duplex rates."""
import json
import os
import time

import torch

out = {"nproc": os.cpu_count(), "meminfo": open("/proc/meminfo").read().splitlines()[:3]}
dev = torch.device("cuda:0")
GB = 1 << 30
sizes = [int(os.environ.get("PROBE_K_GB", "72")), int(os.environ.get("PROBE_V_GB", "31"))]
t = time.perf_counter()
hk = torch.empty(sizes[0] * GB, dtype=torch.uint8, pin_memory=True)
out["pin_K_s"] = time.perf_counter() - t
t = time.perf_counter()
hv = torch.empty(sizes[1] * GB, dtype=torch.uint8, pin_memory=True)
out["pin_V_s"] = time.perf_counter() - t
dk = torch.empty(sizes[0] * GB, dtype=torch.uint8, device=dev)
dv = torch.empty(sizes[1] * GB, dtype=torch.uint8, device=dev)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
for name, pairs in (("h2d", [(dk, hk, s_in)]), ("d2h", [(hv, dv, s_out)]),
                    ("duplex", [(dk, hk, s_in), (hv, dv, s_out)])):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for dst, src, st in pairs:
        with torch.cuda.stream(st):
            dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    out[name + "_s"] = dt
    out[name + "_GBps"] = sum(d.numel() for d, _, _ in pairs) / dt / 1e9
out["meminfo_after"] = open("/proc/meminfo").read().splitlines()[:3]
print(json.dumps(out, indent=1))
