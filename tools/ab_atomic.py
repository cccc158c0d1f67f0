"""A/B of the atomic route: k_atomic_staged vs the legacy k_scatter<atomic> (FEA_ATOMIC_LEGACY=1),
both checked against the sorted route (|a-b| <= 1e-12 max(|a|,|b|,1)).

  python tools/ab_atomic.py [--configs 1,2,3] [--runs 5]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3")
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--staged-only", action="store_true")
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(plan, K, v, runs):
    for _ in range(2):
        v.zero_()
        plan.assemble(K, v, strategy="atomic", accumulate=True)
    ms = []
    for _ in range(runs):
        v.zero_()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.assemble(K, v, strategy="atomic", accumulate=True)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return sum(ms) / len(ms), min(ms)


for cfg in [int(c) for c in a.configs.split(",")]:
    conn, nn, d = M.config_mesh(cfg)
    ed = M.element_dofs(conn, d)
    K = fea.fill_seeded_k(conn.shape[0], ed.shape[1], 42)
    out = {"config": cfg, "lib": os.environ.get("FEA_LIB_PATH", "default")}
    ref = None
    for name, legacy in (("legacy", True), ("staged", False)):
        if legacy and a.staged_only:
            continue
        if legacy:
            os.environ["FEA_ATOMIC_LEGACY"] = "1"
        else:
            os.environ.pop("FEA_ATOMIC_LEGACY", None)
        plan = fea.Plan(ed, nn * d, dofs_per_node=d)
        if ref is None:
            ref = plan.assemble(K, strategy="sorted")
        v = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
        avg, mn = timed(plan, K, v, a.runs)
        ok = bool(torch.all((v - ref).abs() <= 1e-12 * torch.maximum(torch.maximum(v.abs(), ref.abs()),
                                                                      torch.ones_like(v))).item())
        out[name] = {"ms_avg": round(avg, 4), "ms_min": round(mn, 4), "within_1e-12": ok,
                     "launches": plan.last_launches}
        del plan, v
    print(json.dumps(out), flush=True)
