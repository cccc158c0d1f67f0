#!/usr/bin/env python
"""Benchmark of the FE assembly hot path (BASELINE.json configs[1] = SURVEY cfg2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--strategy sorted|atomic|colour]
  python bench.py --impl reference ...      # the reference's own CPU assembly, same workload

Workload (per GPU, weak scaling): hex8 64 x 64 x (64*N) elements, d = 3 DOFs per node
(m = 24), element order permuted (seed 7), K = seeded symmetric U[-1,1) (seed 42).
At N = 1 this is exactly BASELINE cfg2 (hex8 64^3). For N > 1 each rank owns the rows of one
64-layer z-slab (row-partitioned assembly): it keeps the elements touching its
rows, builds its row block's pattern and assembles it; no collective on the data path.

A step = one numeric assembly of the whole workload (K resident in HBM, values written).
Per step, untimed: reset for the atomic route (reference semantics, bench.hpp:98-113) and an
L2 flush (256 MiB memset). Timed: CUDA events around the assembly launch(es) on their stream.
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
NXY = 64
NZ_PER_GPU = 64
D = 3
SEED_K = 42
SEED_PERM = 7
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", action="store_true", help="NCCL gather of row blocks to rank 0 (N>1)")
    ap.add_argument("--check", action="store_true",
                    help="with --gather: rank 0 re-assembles the global mesh on its GPU and compares bitwise")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def global_mesh(n_gpus: int):
    from paper_2012_00585_b200 import meshgen as M
    conn, n_nodes = M.hex8_box(NXY, NXY, NZ_PER_GPU * n_gpus)
    conn = M.permute_elements(conn, SEED_PERM)
    return conn, n_nodes


def owned_rows(n_gpus: int, rank: int):
    """z-slab row ownership: node layers [64r, 64(r+1)) (the last rank also owns the top layer)."""
    layer = (NXY + 1) * (NXY + 1)
    n_layers = NZ_PER_GPU * n_gpus + 1
    lb = NZ_PER_GPU * rank
    le = n_layers if rank == n_gpus - 1 else NZ_PER_GPU * (rank + 1)
    return lb * layer * D, le * layer * D


def workload_config(n_gpus: int, E: int, strategy: str, extra=None):
    cfg = {
        "workload": f"BASELINE configs[1] / SURVEY cfg2 per GPU: hex8 {NXY}x{NXY}x{NZ_PER_GPU * n_gpus} "
                    f"elements (= 64^3 per GPU), d=3 (m=24), element order permuted (seed {SEED_PERM}), "
                    f"K symmetric U[-1,1) from seed {SEED_K}, CSR+CRAC (one values kernel serves both)",
        "elements": E,
        "m": 24,
        "strategy": strategy,
        "parallelism": f"row-partitioned z-slabs x{n_gpus}" if n_gpus > 1 else "single GPU",
        "l2": "256 MiB L2 flush between steps (untimed); K (1.21 GB/GPU) and values (0.52 GB/GPU) exceed the 126 MB L2",
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

    conn, n_nodes = global_mesh(N)
    E_glob = conn.shape[0]
    m = 8 * D
    ed = M.element_dofs(conn, D)
    n_rows = n_nodes * D
    rb, re = owned_rows(N, rank)
    t0 = time.perf_counter()
    plan = fea.Plan(ed, n_rows, dofs_per_node=D, row_range=(rb, re), device=dev.index, k_compact=N > 1)
    torch.cuda.synchronize()
    symbolic_ms = (time.perf_counter() - t0) * 1e3
    E_loc = plan.n_elements
    ids = plan.elements() if N > 1 else None
    K = fea.fill_seeded_k(E_loc, m, SEED_K, elem_ids=ids, device=dev.index)
    values = torch.zeros(plan.nnz, dtype=torch.float64, device=dev)
    colour, n_colours = plan.greedy_colouring()
    plan.set_colouring(colour)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    def one(strategy, accumulate):
        plan.assemble(K, values, strategy=strategy, accumulate=accumulate, stream=stream)
        return plan.last_launches

    def timed(strategy, steps, warmup, sampler=None):
        """Per step: untimed reset (atomic/colour) + L2 flush, then events around the assembly."""
        acc = strategy in ("atomic", "colour_passes")  # element-owner routes add into a reset values array;
        # the segmented reductions overwrite (== reset_values + assemble, same bits)
        for _ in range(warmup):
            if acc:
                values.zero_()
            one(strategy, acc)
        if sampler is not None:  # soak so the clock samples see the GPU under this load
            t_end = time.perf_counter() + float(os.environ.get("FEA_BENCH_SOAK_S", "1.5"))
            while time.perf_counter() < t_end:
                for _ in range(20):
                    one(strategy, acc)
                torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        launches = 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(steps):
            if acc:
                values.zero_()
            flush.zero_()
            evs[i][0].record(stream)
            launches += one(strategy, acc)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = [a.elapsed_time(b) for a, b in evs]
        return sum(ms), ms, launches

    results = {}
    for s in ("sorted", "atomic", "colour", "colour_passes"):
        if s == args.strategy:
            continue
        tot, ms, _ = timed(s, max(3, args.steps // 2), args.warmup)
        results[s] = tot / len(ms)
    with ClockSampler(dev.index) as cs:
        total_ms, ms_list, launches = timed(args.strategy, args.steps, args.warmup, sampler=cs)
    clocks = cs.summary()
    results[args.strategy] = total_ms / args.steps

    # max over ranks (device time)
    t = torch.tensor([total_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_max = float(t.item())
    ms_per_step = total_max / args.steps
    entries = E_glob * m * m  # every element-matrix entry assembled exactly once, job-wide
    value = entries / (ms_per_step * 1e-3)

    # roofline of the dominant kernel on this rank: algorithmic bytes / mean launch time
    npe = 8
    min_bytes = 8 * E_loc * m * m + 8 * plan.nnz + 4 * E_loc * npe
    my_ms = total_ms / args.steps
    peak, peak_src = measured_peak_gbs()
    achieved = min_bytes / (my_ms * 1e-3) / 1e9
    kernel_name = {"sorted": "k_gather_slot<3,8> (warp = node, lane = slot, register accumulators)",
                   "atomic": "k_atomic_staged<3,8,u8> (visit-order metadata, cp.async-staged K, RED.E.ADD.F64)",
                   "colour": "k_gather_slot<3,8> (colour-ordered incidences)",
                   "colour_passes": "k_scatter<32,u8,plain> x n_colours"}[args.strategy]
    traffic = profiled_traffic(f"cfg2/{args.strategy}") if N == 1 else None

    # end to end through the public API with HOST buffers (pinned): every step copies its whole
    # K host->device and its whole values array device->host. Headline form: the pipelined
    # batch call (step i's K upload overlaps step i-1's kernel + values download); the
    # one-shot synchronous call is reported beside it.
    e2e = None
    if not args.no_e2e:
        Kh = [torch.empty(K.shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        for k in Kh:
            k.copy_(K)
        vh = [torch.empty(plan.nnz, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        Kh_np, vh_np = [k.numpy() for k in Kh], [v.numpy() for v in vh]
        e2e_steps = max(4, min(args.steps, 12))
        ks = [Kh_np[i % 2] for i in range(e2e_steps)]
        vs = [vh_np[i % 2] for i in range(e2e_steps)]
        plan.assemble_host_batch(ks[:2], vs[:2], strategy=args.strategy, stream=stream)  # warm-up
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        plan.assemble_host_batch(ks, vs, strategy=args.strategy, stream=stream)
        e2e_s = (time.perf_counter() - t1) / e2e_steps
        t1 = time.perf_counter()
        for i in range(3):
            plan.assemble_host(Kh_np[0], vh_np[0], strategy=args.strategy, stream=stream)
        single_s = (time.perf_counter() - t1) / 3
        te = torch.tensor([e2e_s, single_s], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": entries / float(te[0].item()), "unit": UNIT,
               "h2d_bytes_per_step": int(Kh[0].numel() * 8 * N),
               "d2h_bytes_per_step": int(vh[0].numel() * 8 * N),
               "ms_per_step": float(te[0].item()) * 1e3, "steps": e2e_steps,
               "path": "Plan.assemble_host_batch -> fea_assemble_host_batch: per step pinned K H2D, "
                       "assemble, values D2H; step i's upload overlaps step i-1's download",
               "single_call_ms": float(te[1].item()) * 1e3,
               "single_call_value": entries / float(te[1].item())}
        if args.strategy == "sorted":  # the host paths return the device path's bits
            assert np.array_equal(vh_np[0], values.cpu().numpy()), "e2e values differ"
        del Kh, vh, Kh_np, vh_np, ks, vs

    gather_ms = None
    gathered_nnz = None
    check_ok = None
    fused = None
    if args.gather and world > 1:
        from paper_2012_00585_b200.dist import PeerValues, gather_row_blocks
        # (1) assembly, then an NCCL gather of the row blocks to rank 0
        torch.cuda.synchronize()
        dist.barrier()
        tg = time.perf_counter()
        full = gather_row_blocks(values if backend == "nccl" else values.cpu(), root=0)
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - tg) * 1e3
        # (2) fused: every rank assembles its row block straight into rank 0's global values
        # buffer (CUDA IPC peer mapping): the value stores cross NVLink as they are produced
        pv = PeerValues(plan.nnz, dev, root=0)
        fused_ms = []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.assemble_into(K, pv.ptr, strategy=args.strategy, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            dist.barrier()
            fused_ms.append(e0.elapsed_time(e1))
        tf = torch.tensor([min(fused_ms[1:])], dtype=torch.float64, device=red_dev)
        dist.all_reduce(tf, op=dist.ReduceOp.MAX)
        fused = {"ms": float(tf.item()), "path": "Plan.assemble_into(PeerValues.ptr): CUDA IPC mapping of "
                                                 "rank 0's global values; max over ranks of the kernel time"}
        if rank == 0:
            gathered_nnz = int(full.numel())
            fused["equal_to_nccl_gather"] = bool(torch.equal(pv.full[: full.numel()].cpu(), full.cpu()))
            if args.check:
                gplan = fea.Plan(ed, n_rows, dofs_per_node=D, device=dev.index)
                gK = fea.fill_seeded_k(E_glob, m, SEED_K, device=dev.index)
                want = gplan.assemble(gK, strategy=args.strategy if args.strategy == "sorted" else "sorted")
                check_ok = bool(torch.equal(full.to(dev), want)) if args.strategy == "sorted" else None
                del gplan, gK, want
        dist.barrier()
        pv.close()

    cpu_baseline = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu_baseline = cpu_baseline_sample(conn, n_nodes, K)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(N, E_glob, args.strategy, {
                "nnz_per_gpu": plan.nnz, "crac_runs_per_gpu": plan.n_runs, "n_colours": n_colours,
                "symbolic_phase_ms": round(symbolic_ms, 2),
                "plan_metadata_bytes": plan.metadata_bytes}),
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name,
                         "algorithmic_bytes_per_launch": min_bytes,
                         "bytes_formula": "8*E*m^2 (K) + 8*NNZ (values) + 4*E*npe (connectivity)",
                         "peak_source": peak_src, "frac_of_8TBps": achieved / 8000.0},
            "strategies_ms_per_step": {k: round(v, 4) for k, v in results.items()},
            "strategies_entries_per_s": {k: entries / N / (v * 1e-3) * N for k, v in results.items()},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu_baseline,
        }
        if gather_ms is not None:
            line["gather"] = {"ms": gather_ms, "backend": backend, "rows_blocks_nnz_total": gathered_nnz,
                              "bitwise_equal_to_single_gpu": check_ok,
                              "fused_assembly_into_root": fused}
        if backend != "nccl":
            line["note"] = f"functional run over {backend} with {world} ranks on {torch.cuda.device_count()} GPU(s): not a scaling measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_sample(conn, n_nodes, K_dev):
    """The reference library (oracle/_ref) on the host cores, same cfg2 workload, bounded runs."""
    try:
        import oracle
        if oracle.REF_SO.exists():
            Kh = K_dev.cpu().numpy()
            threads = oracle.hardware_threads()
            prob = oracle.RefProblem(conn, n_nodes, D)
            runs = 5
            t = prob.time(Kh, method="spin-vec", fmt="crac", threads=threads, runs=runs)
            t_avg = float(np.mean(t)) * 1e-6
            entries = conn.shape[0] * 24 * 24
            return {"value": entries / t_avg, "unit": UNIT, "cores": threads, "kind": "reference",
                    "method": "assemble_spin_vectorized / CracSpinMatrix (the paper's fastest CPU method)",
                    "ms_per_assembly": t_avg * 1e3,
                    "sample": f"full cfg2 (E={conn.shape[0]}), fea::time_assembly semantics: reset + "
                              f"1 warm-up + {runs} timed runs, K copied per element from a host buffer"}
        # no reference build: the C oracle port, sequential, one assembly
        Kh = K_dev.cpu().numpy()
        from paper_2012_00585_b200 import meshgen as M
        P = oracle.Pattern.build(conn, n_nodes, D)
        ed = M.element_dofs(conn, D)
        t0 = time.perf_counter()
        P.assemble_sequential(ed, Kh)
        dt = time.perf_counter() - t0
        return {"value": conn.shape[0] * 576 / dt, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": "full cfg2, one sequential assembly (oracle port)"}
    except Exception as ex:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation on the host cores
# ---------------------------------------------------------------------------

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    N = world if world > 1 else args.gpus
    conn, n_nodes = global_mesh(N)
    E = conn.shape[0]
    m = 24
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfea_ref.so not built"}))
        return
    threads = oracle.hardware_threads()
    Kh = oracle.fill_k(SEED_K, E, m)
    t0 = time.perf_counter()
    prob = oracle.RefProblem(conn, n_nodes, D)
    setup_s = time.perf_counter() - t0
    for _ in range(max(0, args.warmup - 1)):
        prob.assemble(Kh, method="spin-vec", fmt="crac", threads=threads)
    t = prob.time(Kh, method="spin-vec", fmt="crac", threads=threads, runs=args.steps)
    t_avg = float(np.mean(t)) * 1e-6
    value = E * m * m / t_avg
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_avg * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(N, E, "reference assemble_spin_vectorized on CracSpinMatrix", {
            "reference_method": "spin-vec/crac (paper's fastest CPU method)",
            "t_min_ms": float(np.min(t)) * 1e-3, "build_pattern_s": setup_s}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"full workload, fea::time_assembly: 1 warm-up + {args.steps} timed runs"},
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
