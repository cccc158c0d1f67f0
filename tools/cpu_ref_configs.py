"""The reference's own CPU assembly methods timed on BASELINE configs 1-4 on this host (the
per-config CPU column beside tools/bench_configs.py's GPU table; reported baseline only).

  python tools/cpu_ref_configs.py [--configs 1,2,3,4] [--runs 3] [--seq-runs 1]

Runs the UNMODIFIED reference library (oracle/_ref/libfea_ref.so, built by
__graft_entry__.build()) through fea::time_assembly semantics (bench.hpp:98-113: untimed reset,
one warm-up, `runs` timed assemblies; t_avg / t_min as bench.cpp:223-224): assemble_sequential on
one thread, assemble_atomic / assemble_spin_vectorized / assemble_coloured_vectorized with every
host thread (fea::default_thread_count, FEA_THREADS honoured), CSR and CRAC targets as the paper
pairs them. K is the same seeded symmetric U[-1,1) matrix the GPU runs use, materialized in host
memory; the supplier copies each element's block (the paper re-creates a ones matrix instead).
Also reports the reference's single-threaded build_pattern time (the symbolic phase).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import oracle  # noqa: E402  (test infrastructure: the reference library is the measured arm here)
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

METHODS = [("seq", "csr", 1), ("atomic", "csr", 0), ("spin-vec", "crac", 0), ("colour-vec", "crac", 0)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--seq-runs", type=int, default=1)
    a = ap.parse_args()
    threads = oracle.hardware_threads()
    for cfg in [int(c) for c in a.configs.split(",")]:
        conn, nn, d = M.config_mesh(cfg)
        E, m = conn.shape[0], conn.shape[1] * d
        t0 = time.perf_counter()
        pr = oracle.RefProblem(conn, nn, d)
        t_pat = time.perf_counter() - t0
        K = oracle.fill_k(M.SEED_K, E, m)
        col, ncol = pr.greedy_colouring(E)
        out = {"config": cfg, "elements": E, "m": m, "nnz": pr.nnz, "host_threads": threads,
               "build_pattern_s": round(t_pat, 3), "n_colours": ncol, "methods": {}}
        for method, fmt, thr in METHODS:
            t = pr.time(K, method=method, fmt=fmt, threads=thr or threads,
                        colour_of=col if method == "colour-vec" else None,
                        runs=a.seq_runs if method == "seq" else a.runs)
            ms = t / 1e3
            out["methods"][f"{method}/{fmt}"] = {
                "threads": thr or threads, "ms_avg": round(float(ms.mean()), 3), "ms_min": round(float(ms.min()), 3),
                "entries_per_s": E * m * m / (float(ms.mean()) / 1e3)}
        print(json.dumps(out), flush=True)
        del pr, K


if __name__ == "__main__":
    main()
