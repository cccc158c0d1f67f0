"""BASELINE config 5 as a row-partitioned (strong-scaling) run: hex8 n^3 (default 256), d = 3,
split into N z-slabs of node rows, one rank per GPU.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29571 tools/cfg5_ranks.py [--size 256] [--gather] [--check]

Each rank builds its plan for its owned rows (elements touching them kept on the device,
FEA_PLAN_K_COMPACT), generates only its kept elements' K, and times the sorted and atomic routes
(CUDA events, barrier on both sides, max over ranks). The whole job's entries/s counts every
element-matrix entry of the global mesh once; the redundant (halo) element work is reported.
--gather: the fused assembly-into-root over peer memory (dist.PeerValues), and with --check the
root compares the gathered values bitwise with a single-plan assembly of the whole mesh (small n).
FEA_BENCH_BACKEND=gloo runs the ranks on fewer GPUs for a functional check (not a measurement).
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=256, help="elements per edge (hex8 size^3)")
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--gather", action="store_true")
ap.add_argument("--check", action="store_true")
a = ap.parse_args()

rank, world, local = (int(os.environ.get(k, v)) for k, v in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
backend = os.environ.get("FEA_BENCH_BACKEND", "nccl")
dev = torch.device("cuda", local % torch.cuda.device_count())
torch.cuda.set_device(dev)
if world > 1:
    dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
red_dev = dev if backend == "nccl" else torch.device("cpu")

n, d = a.size, 3
conn, nn = M.hex8_structured(n)
ed = M.element_dofs(conn, d)
E, m = ed.shape
layer = (n + 1) * (n + 1)
lo = (n + 1) * rank // world
hi = (n + 1) * (rank + 1) // world
plan = fea.Plan(ed, nn * d, dofs_per_node=d, row_range=(lo * layer * d, hi * layer * d), device=dev.index,
                k_compact=world > 1)
E_loc = plan.n_elements
K = fea.fill_seeded_k(E_loc, m, 42, elem_ids=plan.elements() if world > 1 else None, device=dev.index)
values = torch.empty(plan.nnz, dtype=torch.float64, device=dev)


def barrier():
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()


def max_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(strategy):
    acc = strategy != "sorted"
    ms = []
    for i in range(a.runs + 1):
        if acc:
            values.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.assemble(K, values, strategy=strategy, accumulate=acc)
        e1.record()
        barrier()
        if i:
            ms.append(e0.elapsed_time(e1))
    return max_over_ranks(float(np.mean(ms)))


entries = E * m * m
kept = torch.tensor([E_loc], dtype=torch.float64, device=red_dev)
if world > 1:
    dist.all_reduce(kept)
out = {"config": 5, "n": n, "ranks": world, "backend": backend if world > 1 else None, "elements": E,
       "redundant_element_fraction": float(kept.item()) / E - 1.0, "strategies": {}}
for s in ("sorted", "atomic"):
    t = timed(s)
    out["strategies"][s] = {"ms_max_over_ranks": round(t, 3), "entries_per_s": entries / (t * 1e-3)}

if a.gather and world > 1:
    from paper_2012_00585_b200.dist import PeerValues
    pv = PeerValues(plan.nnz, dev, root=0)
    ms = []
    for i in range(a.runs + 1):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.assemble_into(K, pv.ptr, strategy="sorted")
        e1.record()
        barrier()
        if i:
            ms.append(e0.elapsed_time(e1))
    out["fused_assembly_into_root_ms"] = max_over_ranks(float(np.mean(ms)))
    if rank == 0 and a.check:
        gplan = fea.Plan(ed, nn * d, dofs_per_node=d, device=dev.index)
        want = gplan.assemble(fea.fill_seeded_k(E, m, 42, device=dev.index), strategy="sorted")
        out["gathered_bitwise_equal_to_single_plan"] = bool(torch.equal(pv.full, want))
        del gplan, want
    barrier()
    pv.close()

if rank == 0:
    print(json.dumps(out), flush=True)
if world > 1:
    dist.destroy_process_group()
