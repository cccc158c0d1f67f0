"""BASELINE config 5 on ONE B200: hex8 256^3, d=3 — NNZ 4,092,809,481 (> 2^31, int64 offsets),
K 77.3 GB + values 32.7 GB resident. Times the sorted and atomic routes and checks, at full size:
  * NNZ and CRAC runs equal the closed forms; 4096 sampled node rows equal the geometric
    3x3x3 neighbourhood (pattern bit-exactness on a sample, the full CSR is 33 GB);
  * ones-K: sum(values) == E*m^2 exactly, sorted and atomic bitwise equal;
  * seeded K: atomic within 1e-12 (reference tolerance form) of sorted, compared in chunks.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

n, d = 256, 3
t0 = time.perf_counter()
conn, nn = M.hex8_structured(n)
ed = M.element_dofs(conn, d)
E, m = ed.shape
out = {"config": 5, "elements": E, "m": m, "meshgen_s": round(time.perf_counter() - t0, 1)}
torch.cuda.synchronize()
t0 = time.perf_counter()
plan = fea.Plan(ed, nn * d, dofs_per_node=d)
torch.cuda.synchronize()
out["symbolic_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
del ed
out["nnz"] = plan.nnz
out["crac_runs"] = plan.n_runs
out["nnz_closed_form"] = plan.nnz == M.closed_form_nnz("hex8", n, d)
out["runs_closed_form"] = plan.n_runs == d * (n + 1) * (3 * n + 1) ** 2
out["plan_metadata_bytes"] = plan.metadata_bytes

# sampled rows vs the geometric neighbourhood (pattern check without a 33 GB host copy)
rp = torch.empty(plan.n_rows + 1, dtype=torch.int64, device="cuda")
cols = torch.empty(plan.nnz, dtype=torch.int64, device="cuda")
plan._lib.fea_plan_copy_csr(plan._h, fea.assembly._ptr(rp), fea.assembly._ptr(cols))
torch.cuda.synchronize()
rng = np.random.default_rng(5)
nv = n + 1
ok = True
for v in rng.integers(0, nn, size=4096):
    z, y, x = v // (nv * nv), (v // nv) % nv, v % nv
    nb = sorted(((zz * nv + yy) * nv + xx) for zz in range(max(z - 1, 0), min(z + 2, nv))
                for yy in range(max(y - 1, 0), min(y + 2, nv)) for xx in range(max(x - 1, 0), min(x + 2, nv)))
    want = np.array([u * d + k for u in nb for k in range(d)], np.int64)
    for k in range(d):
        r = v * d + k
        a, b = int(rp[r]), int(rp[r + 1])
        ok &= np.array_equal(cols[a:b].cpu().numpy(), want)
out["sampled_rows_match_geometry"] = bool(ok)
del rp, cols
torch.cuda.empty_cache()

K = fea.fill_seeded_k(E, m, 42)
values = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
entries = E * m * m
min_bytes = 8 * entries + 8 * plan.nnz + 4 * E * 8


def timed(strategy, runs=3):
    acc = strategy != "sorted"
    ms = []
    for i in range(runs + 1):
        if acc:
            values.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.assemble(K, values, strategy=strategy, accumulate=acc)
        b.record()
        torch.cuda.synchronize()
        if i:
            ms.append(a.elapsed_time(b))
    avg = float(np.mean(ms))
    return {"ms_avg": round(avg, 3), "entries_per_s": entries / (avg * 1e-3),
            "alg_GBps": round(min_bytes / (avg * 1e-3) / 1e9, 1)}


out["strategies"] = {"sorted": timed("sorted"), "atomic": timed("atomic")}
# seeded K: atomic vs sorted, chunked comparison (a second values array fits: 77 + 2x32.7 GB)
plan.assemble(K, values, strategy="sorted")
ref = values.clone()
plan.assemble(K, values, strategy="atomic")
close = True
CH = 1 << 27
for i in range(0, plan.nnz, CH):
    a, b = values[i:i + CH], ref[i:i + CH]
    close &= bool(torch.all((a - b).abs() <= 1e-12 * torch.maximum(torch.maximum(a.abs(), b.abs()),
                                                                  torch.ones_like(a))).item())
out["atomic_within_1e-12_of_sorted"] = close
del ref
torch.cuda.empty_cache()
# ones: exact conservation, sorted == atomic bitwise
K.fill_(1.0)
plan.assemble(K, values, strategy="sorted")
s_sorted = float(values.sum().item())
ones_sorted = values.clone()
plan.assemble(K, values, strategy="atomic")
out["ones_conservation_exact"] = s_sorted == float(entries)
out["ones_sorted_equals_atomic"] = bool(torch.equal(values, ones_sorted))
print(json.dumps(out), flush=True)
