#!/usr/bin/env python
"""Benchmark of the FE assembly hot path on BASELINE config 5.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--strategy sorted|atomic|colour|colour_passes]
  python bench.py --impl reference ...      # the reference's own CPU assembly, same workload

Workload: BASELINE configs[4] — hex8 256^3 elements (16,777,216), lexicographic element order,
d = 3 DOFs per node (m = 24), K seeded symmetric U[-1,1) (seed 42), CSR + CRAC (one values
kernel serves both): NNZ 4,092,809,481 (> 2^31, int64 value offsets), K 77.3 GB + values
32.7 GB resident in HBM on one B200. The metric is quoted "at 1/2/4/8 GPU" on this config, so:

  N = 1   the whole mesh on one GPU;
  N > 1   strong scaling, row-partitioned: rank r owns a contiguous node range
          (cut at the quantiles of the per-node incidence counts), keeps the elements touching
          it (device compaction), builds its row block's pattern and assembles it with its own
          K slab; no collective on the data path (--gather adds the optional gather to rank 0).

A step = one numeric assembly of the whole job (fea::time_assembly semantics, bench.hpp:98-113:
reset untimed, CUDA events around the assembly). Per step, untimed: the reset for the
element-owner routes and a 256 MiB L2 flush (K and values exceed the 126 MB L2 ~900x anyway).
`value` = element-matrix entries of the whole job / max-over-ranks step time.
`e2e`   = the same assembly through the public host API (Plan.assemble_host ->
fea_assemble_host): per step the whole K goes host->device from pinned memory and the whole
values array comes back device->host (pipelined in windows, see numeric.cu).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "element-matrix entries assembled/sec and achieved HBM GB/s (% of roofline) at 1/2/4/8 GPU"
UNIT = "entries/s"
D = 3
NPE = 8
M_ = D * NPE
SEED_K = 42
SOAK_S = float(os.environ.get("FEA_BENCH_SOAK_S", "0"))
CLOCK_QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="sorted", choices=["sorted", "atomic", "colour", "colour_passes"])
    ap.add_argument("--size", type=int, default=256, help="hex8 size^3 (BASELINE config 5: 256)")
    ap.add_argument("--sample-layers", type=int, default=0,
                    help="CPU legs: element z-layers of the sample (default size/8: the N=8 rank slab)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra-strategies", action="store_true")
    ap.add_argument("--gather", action="store_true", help="N>1: gather row blocks to rank 0 (NCCL + fused IPC)")
    ap.add_argument("--check", action="store_true",
                    help="with --gather: rank 0 compares the gathered values with a single-plan assembly")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload_name(n: int) -> str:
    tag = "BASELINE configs[4] / SURVEY cfg5" if n == 256 else f"config 5 shape at n={n}"
    return (f"{tag}: hex8 {n}^3 elements, d=3 (m=24), lexicographic element order, K symmetric U[-1,1) "
            f"from seed {SEED_K}, CSR+CRAC (one values kernel serves both)")


def workload_config(n: int, n_gpus: int, strategy: str, extra=None):
    cfg = {
        "workload": workload_name(n),
        "elements": n ** 3,
        "m": M_,
        "strategy": strategy,
        "parallelism": (f"row-partitioned x{n_gpus} (contiguous node ranges balanced by incidences, "
                        f"strong scaling)" if n_gpus > 1 else "single GPU"),
        "l2": "256 MiB L2 flush between steps (untimed); K and values exceed the 126 MB L2",
    }
    if extra:
        cfg.update(extra)
    return cfg


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the measured window."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={CLOCK_QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                rows.append(dict(sm=float(f[1]), smax=float(f[2]), power=float(f[3]), util=float(f[4]),
                                 hw=f[6], hwt=f[7], swt=f[8], swp=f[9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [r for r in rows if r["util"] >= 50] or rows
        reasons = set()
        for r in loaded:
            for key, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"),
                              ("swt", "sw_thermal_slowdown"), ("swp", "sw_power_cap")):
                if r[key].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in loaded),
                "sm_max_mhz": max(r["smax"] for r in rows),
                "power_w_max": max(r["power"] for r in rows),
                "samples": len(rows), "samples_under_load": len([r for r in rows if r["util"] >= 50]),
                "reasons": sorted(reasons)}


def measured_peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_traffic(kernel_key: str):
    """DRAM bytes per launch from the committed ncu --set full summary, if present."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(kernel_key)
        except Exception:
            return None
    return None


def rank_nodes(conn, n_nodes: int, world: int, rank: int):
    """Contiguous node range of `rank`, balanced by incidences per node (the K row blocks a
    node's rows gather = the dominant traffic), SURVEY.md §8e."""
    from paper_2012_00585_b200.dist import owned_node_range
    if world == 1:
        return 0, n_nodes
    w = np.bincount(conn.ravel(), minlength=n_nodes)
    return owned_node_range(n_nodes, world, rank, weights=w)


KERNEL_NAMES = {
    "sorted": "k_gather_slot<3,8> (warp = node, lane = slot, register accumulators, TMA bulk copies)",
    "atomic": "k_atomic_patch<3,8,8,4> (2x2x2 element patches pre-reduced in shared memory, TMA bulk staging, "
              "one RED.E.ADD.F64 per distinct slot, patches by ticket in a tiled order)",
    "colour": "k_gather_slot<3,8> (colour-ordered incidences)",
    "colour_passes": "k_scatter<32,u8,plain> x n_colours",
}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2012_00585_b200 as fea
    from paper_2012_00585_b200 import meshgen as M

    rank, world, local = dist_env()
    N = world
    # one process per GPU; FEA_BENCH_BACKEND=gloo lets N ranks share fewer GPUs for a
    # functional check of this path (timings from such a run are not scaling numbers)
    backend = os.environ.get("FEA_BENCH_BACKEND", "nccl")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    red_dev = dev if backend == "nccl" else torch.device("cpu")

    def max_over_ranks(*xs):
        t = torch.tensor(list(xs), dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]

    def sum_over_ranks(*xs):
        t = torch.tensor(list(xs), dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t)
        return [float(v) for v in t.tolist()]

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    n = args.size
    t0 = time.perf_counter()
    conn, n_nodes = M.hex8_structured(n)
    lo, hi = rank_nodes(conn, n_nodes, N, rank)
    ed = M.element_dofs(conn, D)
    E_glob = conn.shape[0]
    meshgen_s = time.perf_counter() - t0
    # CUDA context and kernel images before the symbolic phase is timed (a tiny plan and one
    # assembly of it): neither is part of the phase
    torch.zeros(1, device=dev)
    wc, wn = M.hex8_structured(4)
    with fea.Plan(M.element_dofs(wc, D), wn * D, dofs_per_node=D, device=dev.index) as wplan:
        wplan.assemble(fea.fill_seeded_k(wc.shape[0], M_, SEED_K, device=dev.index))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = fea.Plan(ed, n_nodes * D, dofs_per_node=D, row_range=(lo * D, hi * D), device=dev.index,
                    k_compact=N > 1)
    torch.cuda.synchronize()
    symbolic_ms = (time.perf_counter() - t0) * 1e3
    # the same phase with the element DOFs already on the device (no pageable upload in it)
    ed_dev = torch.from_numpy(ed).to(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan2 = fea.Plan(ed_dev, n_nodes * D, dofs_per_node=D, row_range=(lo * D, hi * D), device=dev.index,
                     k_compact=N > 1)
    torch.cuda.synchronize()
    symbolic_device_ms = (time.perf_counter() - t0) * 1e3
    assert plan2.nnz == plan.nnz
    plan2.close()
    del ed, ed_dev, plan2
    E_loc = plan.n_elements
    ids = plan.elements() if N > 1 else None
    K = fea.fill_seeded_k(E_loc, M_, SEED_K, elem_ids=ids, device=dev.index)
    values = torch.zeros(plan.nnz, dtype=torch.float64, device=dev)
    n_colours = None
    if args.strategy.startswith("colour") or not args.no_extra_strategies:
        t1 = time.perf_counter()
        colour, n_colours = plan.greedy_colouring()
        plan.set_colouring(colour)
        colouring_s = time.perf_counter() - t1
        del colour
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    def timed(strategy, steps, warmup, sampler=None):
        """Per step: untimed reset (element-owner routes) + L2 flush, events around the assembly."""
        acc = strategy in ("atomic", "colour_passes")  # the segmented reductions overwrite
        for _ in range(warmup):
            if acc:
                values.zero_()
            plan.assemble(K, values, strategy=strategy, accumulate=acc, stream=stream)
        # optional soak (FEA_BENCH_SOAK_S seconds of the same load before the timed steps): the
        # sustained, power-capped state instead of the W warm-up + K timed steps of the contract
        if sampler is not None and SOAK_S > 0:
            t_end = time.perf_counter() + SOAK_S
            while time.perf_counter() < t_end:
                for _ in range(4):
                    plan.assemble(K, values, strategy=strategy, accumulate=acc, stream=stream)
                torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        launches = 0
        barrier()
        for i in range(steps):
            if acc:
                values.zero_()
            flush.zero_()
            evs[i][0].record(stream)
            plan.assemble(K, values, strategy=strategy, accumulate=acc, stream=stream)
            launches += plan.last_launches
            evs[i][1].record(stream)
        barrier()
        ms = [a.elapsed_time(b) for a, b in evs]
        return ms, launches

    results = {}
    if not args.no_extra_strategies:
        for s in ("sorted", "atomic", "colour", "colour_passes"):
            if s == args.strategy:
                continue
            ms, _ = timed(s, max(3, args.steps // 4), 2)
            results[s] = max_over_ranks(sum(ms) / len(ms))[0]
    with ClockSampler(dev.index) as cs:
        ms_list, launches = timed(args.strategy, args.steps, args.warmup, sampler=cs)
    clocks = cs.summary()
    my_ms = sum(ms_list) / len(ms_list)
    ms_per_step, t_min_max = max_over_ranks(my_ms, min(ms_list))
    results[args.strategy] = ms_per_step
    entries = E_glob * M_ * M_  # every element-matrix entry of the global mesh, once
    value = entries / (ms_per_step * 1e-3)

    # device result fingerprint (sorted route: the e2e values must equal it bit for bit)
    plan.assemble(K, values, strategy="sorted", stream=stream)
    torch.cuda.synchronize()
    SAMPLE_STRIDE = 4099
    dev_sample = values[::SAMPLE_STRIDE].cpu().numpy().copy()
    dev_sum = int(values.view(torch.int64).sum().item())

    # roofline of the dominant kernel: algorithmic bytes / its mean launch time (per GPU)
    min_bytes_loc = 8 * E_loc * M_ * M_ + 8 * plan.nnz + 4 * E_loc * NPE
    bytes_sum, kept_sum = sum_over_ranks(min_bytes_loc, E_loc)
    peak, peak_src = measured_peak_gbs()
    achieved = bytes_sum / N / (ms_per_step * 1e-3) / 1e9
    traffic = profiled_traffic(f"cfg5/{args.strategy}") if N == 1 and n == 256 else None

    # end to end through the public host API: per step the whole K (pinned host) goes in and
    # the whole values array comes back. Config 5 needs the GPU memory of the device-resident
    # run for its staging, so the device K / values are released first.
    e2e = None
    if not args.no_e2e:
        from paper_2012_00585_b200.hostmem import pinned_empty
        tp = time.perf_counter()
        Kh = pinned_empty((E_loc, M_, M_), np.float64)
        vh = pinned_empty((plan.nnz,), np.float64)
        pin_s = time.perf_counter() - tp
        torch.from_numpy(Kh).copy_(K)
        del K, values
        torch.cuda.empty_cache()
        plan.assemble_host(Kh, vh, strategy=args.strategy, stream=stream)  # warm-up: staging allocation
        barrier()
        times = []
        e2e_launches = 0
        for _ in range(args.e2e_steps):
            barrier()
            t1 = time.perf_counter()
            plan.assemble_host(Kh, vh, strategy=args.strategy, stream=stream)
            times.append(time.perf_counter() - t1)
            e2e_launches += plan.last_launches
        e2e_s, e2e_min_s = max_over_ranks(sum(times) / len(times), min(times))
        same = None
        if args.strategy == "sorted":  # the host path returns the device path's bits
            ok = bool(np.array_equal(vh[::SAMPLE_STRIDE], dev_sample)) and \
                int(vh.view(np.int64).sum(dtype=np.int64)) == dev_sum
            same = max_over_ranks(0.0 if ok else 1.0)[0] == 0.0
        h2d, d2h = sum_over_ranks(Kh.nbytes, vh.nbytes)
        e2e = {"value": entries / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3, "ms_min": e2e_min_s * 1e3,
               "steps": args.e2e_steps, "warmup": 1, "gpu_launches": e2e_launches,
               "path": "Plan.assemble_host -> fea_assemble_host: pinned K host->device in the chunks each "
                       "traversal window needs, windows launched as their chunk lands, each window's values "
                       "range device->host as it completes (H2D, kernels and D2H overlap)",
               "pcie_floor_ms": max(Kh.nbytes, vh.nbytes) / 55e9 * 1e3,
               "pin_s": round(pin_s, 1),
               "values_equal_device_run": same}
        del Kh, vh

    gather = None
    if args.gather and world > 1:
        gather = run_gather(args, plan, dev, backend, M, fea, conn, n_nodes, E_glob, stream)

    cpu_baseline = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu_baseline = cpu_baseline_sample(n, args.sample_layers or max(1, n // 8))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "t_min_ms": t_min_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded structured hex8 mesh and element matrices)",
            "config": workload_config(n, N, args.strategy, {
                "nnz": plan.nnz if N == 1 else None, "nnz_rank0": plan.nnz,
                "crac_runs_rank0": plan.n_runs, "n_colours": n_colours,
                "redundant_element_fraction": kept_sum / E_glob - 1.0,
                "meshgen_s": round(meshgen_s, 2), "soak_s": SOAK_S, "symbolic_phase_ms_rank0": round(symbolic_ms, 1),
                "symbolic_phase_device_dofs_ms_rank0": round(symbolic_device_ms, 1),
                "plan_metadata_bytes_rank0": plan.metadata_bytes}),
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": KERNEL_NAMES[args.strategy],
                         "algorithmic_bytes_per_launch": bytes_sum / N,
                         "bytes_formula": "8*E*m^2 (K) + 8*NNZ (values) + 4*E*npe (connectivity), per GPU",
                         "peak_source": peak_src, "frac_of_8TBps": achieved / 8000.0},
            "strategies_ms_per_step": {k: round(v, 4) for k, v in results.items()},
            "strategies_entries_per_s": {k: entries / (v * 1e-3) for k, v in results.items()},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu_baseline,
        }
        if gather is not None:
            line["gather"] = gather
        if backend != "nccl" and world > 1:
            line["note"] = (f"functional run over {backend} with {world} ranks on {torch.cuda.device_count()} "
                            f"GPU(s): not a scaling measurement")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_gather(args, plan, dev, backend, M, fea, conn, n_nodes, E_glob, stream):
    """N>1 extras: (1) NCCL gather of the row blocks to rank 0 after the assembly; (2) the fused
    form — every rank assembles its row block straight into rank 0's global values buffer mapped
    over CUDA IPC (value stores cross NVLink as they are produced). K is regenerated (the e2e
    leg released it)."""
    import torch
    import torch.distributed as dist
    from paper_2012_00585_b200.dist import PeerValues, gather_row_blocks
    rank = dist.get_rank()
    ids = plan.elements()
    K = fea.fill_seeded_k(plan.n_elements, M_, SEED_K, elem_ids=ids, device=dev.index)
    values = plan.assemble(K, strategy="sorted", stream=stream)
    torch.cuda.synchronize()
    dist.barrier()
    tg = time.perf_counter()
    full = gather_row_blocks(values if backend == "nccl" else values.cpu(), root=0)
    torch.cuda.synchronize()
    gather_ms = (time.perf_counter() - tg) * 1e3
    del values
    torch.cuda.empty_cache()
    pv = PeerValues(plan.nnz, dev, root=0)
    fused_ms = []
    for _ in range(3):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.assemble_into(K, pv.ptr, strategy="sorted", stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        fused_ms.append(e0.elapsed_time(e1))
    red = dev if backend == "nccl" else torch.device("cpu")
    tf = torch.tensor([min(fused_ms[1:]), gather_ms], dtype=torch.float64, device=red)
    dist.all_reduce(tf, op=dist.ReduceOp.MAX)
    out = {"nccl_gather_ms": float(tf[1]), "backend": backend,
           "fused_assembly_into_root_ms": float(tf[0]),
           "path": "Plan.assemble_into(PeerValues.ptr): CUDA IPC mapping of rank 0's global values; "
                   "max over ranks of the kernel time"}
    if rank == 0:
        out["rows_blocks_nnz_total"] = int(full.numel())
        out["fused_equal_to_nccl_gather"] = bool(torch.equal(pv.full[: full.numel()].to(full.device), full))
        if args.check:
            ed = M.element_dofs(conn, D)
            gplan = fea.Plan(ed, n_nodes * D, dofs_per_node=D, device=dev.index)
            want = gplan.assemble(fea.fill_seeded_k(E_glob, M_, SEED_K, device=dev.index), strategy="sorted")
            out["bitwise_equal_to_single_gpu"] = bool(torch.equal(full.to(dev), want))
            del gplan, want
    dist.barrier()
    pv.close()
    del K
    return out


# ---------------------------------------------------------------------------
# CPU legs: the reference library (oracle/_ref) on a bounded sample of the same workload
# ---------------------------------------------------------------------------

REF_METHODS = (("spin-vec", "crac"), ("colour-vec", "crac"), ("atomic", "csr"), ("seq", "csr"))


def reference_sample(n: int, layers: int):
    """The first `layers` element z-layers of config 5 (element ids 0 .. n*n*layers-1, the same
    seeded K): a z-slab of the workload, the size of one rank's share at N = n/layers."""
    import oracle
    from paper_2012_00585_b200 import meshgen as M
    conn, n_nodes = M.hex8_box(n, n, layers)
    t0 = time.perf_counter()
    Kh = oracle.fill_k(SEED_K, conn.shape[0], M_)
    fill_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    prob = oracle.RefProblem(conn, n_nodes, D)
    pattern_s = time.perf_counter() - t0
    return conn, Kh, prob, {"fill_k_s": round(fill_s, 1), "build_pattern_s": round(pattern_s, 1)}


def time_methods(prob, conn, Kh, threads, runs, seq_runs=1):
    """fea::time_assembly (bench.hpp:98-113) of the reference's four assembly methods (the
    bench's method set, bench.cpp:126-156); t_avg / t_min as the reference reports them
    (bench.cpp:223-224). seq runs on 1 thread, the others on `threads`."""
    col, nc = prob.greedy_colouring(conn.shape[0])
    out = {}
    for meth, fmt in REF_METHODS:
        thr = 1 if meth == "seq" else threads
        t = prob.time(Kh, method=meth, fmt=fmt, threads=thr,
                      colour_of=col if meth == "colour-vec" else None, runs=seq_runs if meth == "seq" else runs)
        out[f"{meth}/{fmt}"] = {"t_avg_ms": float(np.mean(t)) * 1e-3, "t_min_ms": float(np.min(t)) * 1e-3,
                                "threads": thr, "runs": len(t)}
    return out, col, nc


def cpu_baseline_sample(n: int, layers: int):
    """cpu_baseline of our line: the reference library, host cores, bounded sample."""
    try:
        import oracle
        if not oracle.REF_SO.exists():
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref/libfea_ref.so missing"}
        threads = oracle.hardware_threads()
        conn, Kh, prob, setup = reference_sample(n, layers)
        methods, _, nc = time_methods(prob, conn, Kh, threads, runs=3)
        best = min((k for k in methods if not k.startswith("seq")), key=lambda k: methods[k]["t_avg_ms"])
        entries = conn.shape[0] * M_ * M_
        return {"value": entries / (methods[best]["t_avg_ms"] * 1e-3), "unit": UNIT, "cores": threads,
                "kind": "reference", "method": best, "methods": methods, "n_colours": nc, **setup,
                "sample": f"first {layers} element z-layers of the workload (hex8 {n}x{n}x{layers}, "
                          f"E={conn.shape[0]}, element ids 0..E-1, same seeded K), fea::time_assembly: "
                          f"reset + 1 warm-up + 3 timed runs per method (seq: 1), K copied per element "
                          f"from a host buffer by the supplier"}
    except Exception as ex:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (the unmodified library,
    oracle/_ref) on all host threads; rank 0 only under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    N = world if world > 1 else args.gpus
    n = args.size
    layers = args.sample_layers or max(1, n // 8)
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfea_ref.so not built"}))
        return
    threads = oracle.hardware_threads()
    conn, Kh, prob, setup = reference_sample(n, layers)
    E = conn.shape[0]
    methods, col, nc = time_methods(prob, conn, Kh, threads, runs=3)
    best = min((k for k in methods if not k.startswith("seq")), key=lambda k: methods[k]["t_avg_ms"])
    meth, fmt = best.split("/")
    colour = col if meth == "colour-vec" else None
    for _ in range(max(0, args.warmup - 1)):  # time_assembly adds its own warm-up run
        prob.assemble(Kh, method=meth, fmt=fmt, threads=threads, colour_of=colour)
    t = prob.time(Kh, method=meth, fmt=fmt, threads=threads, colour_of=colour, runs=args.steps)
    t_avg = float(np.mean(t)) * 1e-6
    value = E * M_ * M_ / t_avg
    sample = (f"first {layers} element z-layers of the workload (hex8 {n}x{n}x{layers}, E={E}, element ids "
              f"0..E-1, same seeded K); every step one full assembly of the sample")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_avg * 1e3,
        "t_min_ms": float(np.min(t)) * 1e-3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded structured hex8 mesh and element matrices)",
        "config": workload_config(n, N, f"reference {meth} on {'CracSpinMatrix' if meth == 'spin-vec' else fmt}", {
            "reference_method": f"{best} (fastest of the reference's methods on this sample)",
            "methods": methods, "n_colours": nc, **setup}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample + f"; fea::time_assembly: 1 warm-up + {args.steps} timed runs"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _relaunch_under_torchrun(n: int) -> int:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29533"),
           __file__, *sys.argv[1:]]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse_args()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_under_torchrun(a.gpus))
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
