"""Per-stage wall time of the symbolic phase (FEA_PLAN_TRACE) on a BASELINE config, with the
element DOFs in pageable host memory (what bench.py passes) and already on the device.

    python tools/plan_trace.py --config 5
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["FEA_PLAN_TRACE"] = "1"

import torch  # noqa: E402

import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

CONFIGS = {1: ("quad4", 256, None, 1), 2: ("hex8", 64, "elements", 3), 3: ("tet4", 128, "nodes", 1),
           4: ("hex27", 48, None, 3), 5: ("hex8", 256, None, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--lazy", action="store_true", help="time the first call of each route (lazily built tables)")
    a = ap.parse_args()
    kind, n, perm, d = CONFIGS[a.config]
    conn, nn = M.make_mesh(kind, n, perm)
    ed = M.element_dofs(conn, d)
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    for where in ("host", "device"):
        src = ed if where == "host" else torch.from_numpy(ed).cuda()
        for rep in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan = fea.Plan(src, nn * d, dofs_per_node=d, device=0)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
            print(f"cfg{a.config} DOFs on {where} rep {rep}: plan {ms:.1f} ms, nnz {plan.nnz}", file=sys.stderr, flush=True)
            if a.lazy and where == "device" and rep == 0:
                K = fea.fill_seeded_k(conn.shape[0], ed.shape[1], 42)
                v = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
                for strategy in ("sorted", "atomic", "atomic"):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    plan.assemble(K, v, strategy=strategy, accumulate=strategy == "atomic")
                    torch.cuda.synchronize()
                    print(f"cfg{a.config} {strategy} call: {(time.perf_counter() - t0) * 1e3:.1f} ms", file=sys.stderr, flush=True)
                t0 = time.perf_counter()
                col, nc = plan.greedy_colouring()
                t1 = time.perf_counter()
                plan.set_colouring(col)
                torch.cuda.synchronize()
                print(f"cfg{a.config} greedy colouring {(t1 - t0) * 1e3:.1f} ms ({nc} colours), set_colouring "
                      f"{(time.perf_counter() - t1) * 1e3:.1f} ms", file=sys.stderr, flush=True)
                del K, v
            plan.close()
        del src


if __name__ == "__main__":
    main()
