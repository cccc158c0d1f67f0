"""Per-assembly time of back-to-back assemblies replayed from a CUDA graph (the launch-bound
case: config 1 is 14 MB of traffic, ~2 us at the HBM roofline, while one launch from the host
costs ~10 us of launch latency).

  python tools/graph_batch.py [--configs 1,2,3] [--batch 64] [--buffers 16] [--replays 5]

A graph holds `batch` assemblies; assembly i reads K buffer i % buffers and writes values
buffer i % buffers, so the batch's working set (buffers x (K + values)) exceeds the 126 MB L2
and every assembly streams its inputs from HBM. Time = CUDA events around the graph replays;
per-assembly time = total / (replays * batch). Values of the last replay are checked bitwise
against a plain (non-graph) assembly of the same buffer.
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--buffers", type=int, default=16)
ap.add_argument("--replays", type=int, default=5)
ap.add_argument("--strategies", default="sorted,atomic")
ap.add_argument("--branches", type=int, default=1,
                help="independent assemblies run as this many parallel graph branches (fork/join on events)")
a = ap.parse_args()

for cfg in (int(c) for c in a.configs.split(",")):
    conn, nn, d = M.config_mesh(cfg)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    npe = conn.shape[1]
    plan = fea.Plan(ed, nn * d, dofs_per_node=d)
    nb = a.buffers
    Ks = [fea.fill_seeded_k(E, m, 42 + i) for i in range(nb)]
    Vs = [torch.zeros(plan.nnz, dtype=torch.float64, device="cuda") for _ in range(nb)]
    alg = 8 * E * m * m + 8 * plan.nnz + 4 * E * npe
    out = {"config": cfg, "branches": a.branches, "elements": E, "m": m, "nnz": plan.nnz, "algorithmic_bytes": alg,
           "working_set_bytes": nb * (8 * E * m * m + 8 * plan.nnz), "batch": a.batch, "strategies": {}}
    s = torch.cuda.Stream()
    for strategy in a.strategies.split(","):
        acc = strategy == "atomic"
        with torch.cuda.stream(s):
            plan.assemble(Ks[0], Vs[0], strategy=strategy, accumulate=acc, stream=s)  # lazy tables
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = [torch.cuda.Stream() for _ in range(a.branches)]
        with torch.cuda.graph(g, stream=s):
            fork = torch.cuda.Event()
            fork.record(s)
            for b, ss in enumerate(side):  # branch b: assemblies b, b + branches, ...
                ss.wait_event(fork)
                with torch.cuda.stream(ss):
                    for i in range(b, a.batch, a.branches):
                        if acc:
                            Vs[i % nb].zero_()
                        plan.assemble(Ks[i % nb], Vs[i % nb], strategy=strategy, accumulate=acc, stream=ss)
                join = torch.cuda.Event()
                join.record(ss)
                s.wait_event(join)
        with torch.cuda.stream(s):  # replay() launches on the current stream
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.replays):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        per = e0.elapsed_time(e1) / (a.replays * a.batch)
        # check the graph's result (last buffer written) against a plain sorted assembly
        want = torch.zeros_like(Vs[0])
        with torch.cuda.stream(s):
            plan.assemble(Ks[(a.batch - 1) % nb], want, strategy="sorted", stream=s)
        torch.cuda.synchronize()
        got = Vs[(a.batch - 1) % nb]
        same = bool(torch.equal(got, want)) if strategy == "sorted" else \
            bool(torch.all((got - want).abs() <= 1e-12 * torch.maximum(torch.maximum(got.abs(), want.abs()),
                                                                      torch.ones_like(got))).item())
        # plain (non-graph) launches: per-call time including the host launch path
        with torch.cuda.stream(s):
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(s)
            for i in range(a.batch):
                if acc:
                    Vs[i % nb].zero_()
                plan.assemble(Ks[i % nb], Vs[i % nb], strategy=strategy, accumulate=acc, stream=s)
            p1.record(s)
        torch.cuda.synchronize()
        plain = p0.elapsed_time(p1) / a.batch
        out["strategies"][strategy] = {
            "graph_us_per_assembly": round(per * 1e3, 2), "plain_launch_us_per_assembly": round(plain * 1e3, 2),
            "graph_alg_GBps": round(alg / (per * 1e-3) / 1e9, 1), "checked": same,
            "note": "atomic includes the zeroing memset of its values buffer" if acc else ""}
    print(json.dumps(out), flush=True)
    del plan, Ks, Vs
    torch.cuda.empty_cache()
