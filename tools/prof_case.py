"""Small fixed workload for ncu: build a BASELINE config plan and run the numeric kernels a few times.

  python tools/prof_case.py --cfg 2 --strategies sorted,atomic --iters 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--strategies", default="sorted,atomic,colour")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
conn, nn, d = M.config_mesh(a.cfg, a.n)
ed = M.element_dofs(conn, d)
plan = fea.Plan(ed, nn * d, dofs_per_node=d)
K = fea.fill_seeded_k(conn.shape[0], ed.shape[1], 42)
v = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
strategies = a.strategies.split(",")
if "colour" in strategies:
    plan.set_colouring(plan.greedy_colouring()[0])
for s in strategies:
    for _ in range(a.iters):
        if s == "fused":
            plan.assemble_seeded(42, v, strategy="sorted")
        else:
            plan.assemble(K, v, strategy=s, accumulate=s != "sorted")
torch.cuda.synchronize()
print("ok", plan.nnz, plan.n_runs)
