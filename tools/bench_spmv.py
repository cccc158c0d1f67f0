"""SpMV on the assembled matrix: CSR vs CRAC vs node blocks (bytes moved and time).

  python tools/bench_spmv.py [--configs 2,4]
bytes: values 8*nnz + index (CSR 8*nnz int64 cols; CRAC 16*runs + 8*rows; nodes 4*nnz/d^2 +
8*nodes) + x (8*rows, L2) + y (8*rows).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

PEAK = 6552.6
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,4")
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in [int(c) for c in a.configs.split(",")]:
    conn, nn, d = M.config_mesh(cfg)
    ed = M.element_dofs(conn, d)
    plan = fea.Plan(ed, nn * d, dofs_per_node=d)
    K = fea.fill_seeded_k(conn.shape[0], ed.shape[1], 42)
    vals = plan.assemble(K, strategy="sorted")
    del K
    rp = torch.empty(plan.n_rows + 1, dtype=torch.int64, device="cuda")
    cs = torch.empty(plan.nnz, dtype=torch.int64, device="cuda")
    cp = torch.empty(plan.n_rows + 1, dtype=torch.int64, device="cuda")
    ca = torch.empty(2 * plan.n_runs + 2, dtype=torch.int64, device="cuda")
    plan._lib.fea_plan_copy_csr(plan._h, fea.assembly._ptr(rp), fea.assembly._ptr(cs))
    plan._lib.fea_plan_copy_crac(plan._h, fea.assembly._ptr(cp), fea.assembly._ptr(ca))
    x = torch.rand(plan.n_rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    runs = {"csr": lambda: fea.spmv_csr(rp, cs, vals, x, y), "crac": lambda: fea.spmv_crac(cp, ca, vals, x, y),
            "nodes": lambda: plan.spmv(vals, x, y)}
    nb = {"csr": 8 * plan.nnz + 8 * plan.nnz + 8 * (plan.n_rows + 1),
          "crac": 8 * plan.nnz + 16 * plan.n_runs + 8 * (plan.n_rows + 1),
          "nodes": 8 * plan.nnz + 4 * plan.nnz // (d * d) + 8 * (plan.n_rows // d + 1)}
    out = {"config": cfg, "nnz": plan.nnz, "runs": plan.n_runs, "rows": plan.n_rows}
    ref = None
    for name, f in runs.items():
        f()
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        ms = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = float(np.mean(ms))
        byts = nb[name] + 16 * plan.n_rows
        out[name] = {"ms": round(t, 4), "bytes": byts, "GBps": round(byts / t / 1e6, 1),
                     "frac": round(byts / t / 1e6 / PEAK, 3),
                     "max_rel_diff_vs_csr": float(((y - ref).abs() / ref.abs().clamp_min(1e-300)).max())}
    print(json.dumps(out), flush=True)
    plan.close()
    del vals, rp, cs, cp, ca
    torch.cuda.empty_cache()
