"""Quick A/B timer: one strategy on full-size BASELINE configs (L2 flushed, CUDA events), plus a
checksum of the values so variants can be compared for identical bits.

  FEA_LIB_PATH=variants/libfea_x.so python tools/ab_time.py --configs 3,4 --strategy sorted
"""
import argparse
import hashlib
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,4")
ap.add_argument("--strategy", default="sorted")
ap.add_argument("--runs", type=int, default=10)
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in [int(c) for c in a.configs.split(",")]:
    conn, nn, d = M.config_mesh(cfg)
    ed = M.element_dofs(conn, d)
    K = fea.fill_seeded_k(conn.shape[0], ed.shape[1], 42)
    plan = fea.Plan(ed, nn * d, dofs_per_node=d)
    if a.strategy == "colour":
        plan.set_colouring(plan.greedy_colouring()[0])
    v = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
    acc = a.strategy in ("atomic", "colour_passes")
    ms = []
    for i in range(a.runs + 2):
        if acc:
            v.zero_()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.assemble(K, v, strategy=a.strategy, accumulate=acc)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    h = hashlib.sha1(v.cpu().numpy().tobytes()).hexdigest()[:12] if not acc else None
    print(json.dumps({"config": cfg, "lib": os.environ.get("FEA_LIB_PATH", "default"), "strategy": a.strategy,
                      "ms_avg": round(sum(ms) / len(ms), 4), "ms_min": round(min(ms), 4), "sha1": h}), flush=True)
    del plan, v, K
