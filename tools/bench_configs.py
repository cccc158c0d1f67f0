"""All BASELINE configs at full size on one GPU: symbolic-phase time, numeric time per strategy,
entries/s, algorithmic GB/s and roofline fraction, plus size-independent parity properties.

  python tools/bench_configs.py [--configs 1,2,3,4,5] [--runs 5] [--oracle]

Parity at full size (each config): NNZ and CRAC runs equal the closed forms (structured meshes),
ones-K conservation sum(values) == E*m^2 exactly, all three strategies bitwise equal with ones K,
and with random K: atomic and colour within 1e-12 of sorted. --oracle additionally compares the
sorted route bit-for-bit against the CPU oracle's assemble_sequential (configs 1-3).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

PEAK = 6552.6
try:
    PEAK = float(json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:
    pass


def time_strategy(plan, K, values, strategy, runs, flush):
    acc = strategy in ("atomic", "colour_passes")
    for _ in range(2):
        if acc:
            values.zero_()
        plan.assemble(K, values, strategy=strategy, accumulate=acc)
    ms = []
    for _ in range(runs):
        if acc:
            values.zero_()
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.assemble(K, values, strategy=strategy, accumulate=acc)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.mean(ms)), float(np.min(ms)), plan.last_launches


def close(a, b, tol=1e-12):
    return bool(torch.all((a - b).abs() <= tol * torch.maximum(torch.maximum(a.abs(), b.abs()),
                                                               torch.ones_like(a))).item())


def run_config(cfg, runs, use_oracle):
    c = M.CONFIGS[cfg]
    t0 = time.perf_counter()
    conn, nn, d = M.config_mesh(cfg)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    npe = conn.shape[1]
    gen_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ed_dev = torch.from_numpy(ed).cuda()
    plan = fea.Plan(ed_dev, nn * d, dofs_per_node=d)
    torch.cuda.synchronize()
    sym_ms = (time.perf_counter() - t0) * 1e3
    del ed_dev
    t0 = time.perf_counter()
    col, nc = plan.greedy_colouring()
    plan.set_colouring(col)
    col_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, nc_jp = plan.jp_colouring(seed=1)
    jp_ms = (time.perf_counter() - t0) * 1e3
    K = fea.fill_seeded_k(E, m, M.SEED_K)
    values = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    entries = E * m * m
    min_bytes = 8 * entries + 8 * plan.nnz + 4 * E * npe
    out = {"config": cfg, "name": c["name"], "elements": E, "m": m, "rows": plan.n_rows, "nnz": plan.nnz,
           "crac_runs": plan.n_runs, "n_colours": nc, "symbolic_ms": round(sym_ms, 2),
           "colouring_host_s": round(col_s, 3), "jp_colouring_gpu_ms": round(jp_ms, 2), "jp_colours": nc_jp,
           "meshgen_s": round(gen_s, 2),
           "min_bytes": min_bytes, "plan_metadata_bytes": plan.metadata_bytes, "strategies": {}}
    for s in ("sorted", "atomic", "colour", "colour_passes"):
        avg, mn, launches = time_strategy(plan, K, values, s, runs, flush)
        gbs = min_bytes / (avg * 1e-3) / 1e9
        out["strategies"][s] = {"ms_avg": round(avg, 4), "ms_min": round(mn, 4), "launches": launches,
                                "entries_per_s": entries / (avg * 1e-3), "alg_GBps": round(gbs, 1),
                                "frac_measured_peak": round(gbs / PEAK, 4)}
    # fused supplier: K generated inside the gather (no 8*E*m^2 read); bytes = values + connectivity
    ms = []
    for i in range(runs + 1):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.assemble_seeded(M.SEED_K, values, strategy="sorted")
        b.record()
        torch.cuda.synchronize()
        if i:
            ms.append(a.elapsed_time(b))
    fb = 8 * plan.nnz + 4 * E * npe
    avg = float(np.mean(ms))
    out["strategies"]["sorted_fused_supplier"] = {
        "ms_avg": round(avg, 4), "entries_per_s": entries / (avg * 1e-3), "alg_bytes": fb,
        "alg_GBps": round(fb / (avg * 1e-3) / 1e9, 1), "frac_measured_peak": round(fb / (avg * 1e-3) / 1e9 / PEAK, 4)}
    ref = plan.assemble(K, strategy="sorted").clone()
    # ---- parity properties at full size ----
    par = {}
    if True:
        try:
            par["nnz_closed_form"] = plan.nnz == M.closed_form_nnz(c["mesh"], c["n"], d)
        except ValueError:
            pass
    res = {}
    for s in ("sorted", "atomic", "colour", "colour_passes"):
        res[s] = plan.assemble(K, strategy=s).clone()
    par["fused_supplier_bitwise"] = bool(torch.equal(plan.assemble_seeded(M.SEED_K, strategy="sorted"), ref))
    del ref
    par["atomic_within_1e-12"] = close(res["atomic"], res["sorted"])
    par["colour_within_1e-12"] = close(res["colour"], res["sorted"])
    par["colour_passes_bitwise_equal_colour"] = bool(torch.equal(res["colour"], res["colour_passes"]))
    del res
    ones = torch.ones((E, m, m), dtype=torch.float64, device="cuda") if E * m * m * 8 < 40e9 else None
    if ones is not None:
        vo = {s: plan.assemble(ones, strategy=s).clone() for s in ("sorted", "atomic", "colour")}
        par["ones_conservation_exact"] = float(vo["sorted"].sum().item()) == float(entries)
        par["ones_all_strategies_bitwise"] = bool(torch.equal(vo["sorted"], vo["atomic"]) and
                                                 torch.equal(vo["sorted"], vo["colour"]))
        del vo, ones
    if use_oracle and cfg in (1, 2, 3):
        import oracle
        P = oracle.Pattern.build(conn, nn, d)
        rp, cs = plan.csr()
        orp, ocs = P.arrays()
        par["pattern_vs_oracle"] = bool(np.array_equal(rp, orp) and np.array_equal(cs, ocs))
        cp, ca = plan.crac()
        ocp, oca = P.crac()
        par["crac_vs_oracle"] = bool(np.array_equal(cp, ocp) and np.array_equal(ca, oca))
        Kh = K.cpu().numpy()
        want = P.assemble_sequential(ed, Kh)
        got = plan.assemble(K, strategy="sorted").cpu().numpy()
        par["sorted_bitexact_vs_oracle"] = got.tobytes() == want.tobytes()
        ocol, onc = oracle.greedy_colouring(conn, nn)
        par["colouring_vs_oracle"] = bool(np.array_equal(ocol, col))
        got = plan.assemble(K, strategy="colour").cpu().numpy()
        par["colour_bitexact_vs_oracle"] = got.tobytes() == P.assemble_coloured(ed, Kh, ocol).tobytes()
    out["parity"] = par
    plan.close()
    del K, values
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    results = []
    for cfg in [int(x) for x in a.configs.split(",")]:
        r = run_config(cfg, a.runs, a.oracle)
        print(json.dumps(r), flush=True)
        results.append(r)
    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
