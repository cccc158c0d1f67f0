"""How much does the clock sampler itself cost? cfg2 sorted assemblies back to back for ~2 s per
variant: no sampler, nvidia-smi at 100 / 200 / 500 ms (bench.py's query and the recipe's), and
an in-process NVML thread (clocks only / clocks + reasons + power)."""
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

FULL = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
        "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
RECIPE = FULL.replace("utilization.gpu,", "")
conn, nn, d = M.config_mesh(2)
ed = M.element_dofs(conn, d)
K = fea.fill_seeded_k(conn.shape[0], ed.shape[1], 42)
plan = fea.Plan(ed, nn * d, dofs_per_node=d)
v = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")


def run(seconds=2.0):
    for _ in range(20):
        plan.assemble(K, v, strategy="sorted")
    torch.cuda.synchronize()
    n, t0 = 0, time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(50):
            plan.assemble(K, v, strategy="sorted")
        n += 50
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def smi(query, ms):
    return subprocess.Popen(["nvidia-smi", f"--query-gpu={query}", "--format=csv,noheader,nounits", "-lms", str(ms), "-i", "0"],
                            stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


print("none", round(run(), 4), flush=True)
for name, q, ms in (("smi full 100", FULL, 100), ("smi recipe 200", RECIPE, 200), ("smi recipe 500", RECIPE, 500),
                    ("smi clocks-only 100", "index,clocks.sm,clocks.max.sm", 100)):
    p = smi(q, ms)
    time.sleep(0.3)
    print(name, round(run(), 4), flush=True)
    p.terminate()
    p.wait()
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    for name, heavy in (("nvml clocks 50", False), ("nvml clocks+reasons+power 50", True)):
        stop = threading.Event()

        def loop():
            while not stop.is_set():
                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                if heavy:
                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    pynvml.nvmlDeviceGetPowerUsage(h)
                time.sleep(0.05)

        th = threading.Thread(target=loop)
        th.start()
        print(name, round(run(), 4), flush=True)
        stop.set()
        th.join()
except Exception as e:  # noqa: BLE001
    print("pynvml:", e)
print("none again", round(run(), 4), flush=True)
