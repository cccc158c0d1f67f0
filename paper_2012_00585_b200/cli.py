"""Command-line front end over the GPU backend, mirroring the reference's `fea` tool
(proj/tools/fea_main.cpp) so results compare like for like with the reference's outputs.

  python -m paper_2012_00585_b200 assemble --mesh hex8:16 --d 3 --method seq --format crac [--dump A.mtx]
  python -m paper_2012_00585_b200 bench    --mesh gen:256 --methods seq,atomic,colour-vec --runs 30 --out r
  python -m paper_2012_00585_b200 verify   --mesh tet4:6:perm-nodes --d 1
  python -m paper_2012_00585_b200 colour   --mesh hex8:8:perm-elements --out colours.csv

Mesh specs: "gen:N" is the reference's structured n-by-n quad mesh (mesh.cpp:62-85); the 3D
BASELINE meshes are "hex8:N", "tet4:N", "hex27:N", optionally suffixed ":perm-elements" or
":perm-nodes" (seed 7); an ".msh" path is read as ASCII MSH 2.2 (msh.py: quads, tet4, hex8).
p > 1 hierarchical DOF numbering is out of scope.
Methods: seq (the deterministic sort-by-slot route, bit-identical to assemble_sequential),
atomic, colour-vec (bit-identical to assemble_coloured_vectorized under the greedy colouring);
spin and spin-vec have no GPU counterpart. Exit codes as the reference (fea_main.cpp:34-37):
0 ok, 1 usage, 2 verification failed, 3 runtime error.
CSV schemas: bench.cpp:314-335. Matrix Market dump: formats.hpp:366-379.
"""
from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass, field

import numpy as np

from . import meshgen as M

EXIT_OK, EXIT_USAGE, EXIT_VERIFY_FAILED, EXIT_RUNTIME = 0, 1, 2, 3
METHODS = {"seq": "sorted", "atomic": "atomic", "colour-vec": "colour"}
FORMATS = ("csr", "crac")


class UsageError(Exception):
    pass


def parse_mesh(spec: str):
    """-> (label, n, conn, n_nodes). A path to an ASCII MSH 2.2 file is read with msh.import_msh
    (quads, or one volume type: tet4 / hex8); warnings go to stderr like the reference."""
    import os
    if spec.endswith(".msh") or os.path.isfile(spec):
        from . import msh
        try:
            text = open(spec).read()
        except OSError as e:
            raise UsageError(f"cannot read {spec}: {e}") from None
        conn, nn, _, warnings, _ = msh.import_msh(text, kind="auto")
        for w in warnings:
            print(f"warning: {spec}: {w}", file=sys.stderr)
        return spec, 0, conn, nn
    parts = spec.split(":")
    kind = parts[0]
    if kind not in ("gen", "quad4", "hex8", "tet4", "hex27") or len(parts) < 2:
        raise UsageError(f"mesh spec '{spec}': expected gen:N, hex8|tet4|hex27:N[:perm-elements|perm-nodes] "
                         "or an .msh file")
    try:
        n = int(parts[1])
    except ValueError:
        raise UsageError(f"mesh spec '{spec}': n must be an integer") from None
    if n < 1:
        raise UsageError(f"mesh spec '{spec}': n must be >= 1")
    perm = None
    if len(parts) > 2:
        if parts[2] not in ("perm-elements", "perm-nodes"):
            raise UsageError(f"mesh spec '{spec}': unknown modifier '{parts[2]}'")
        perm = parts[2].split("-")[1]
    conn, nn = M.make_mesh("quad4" if kind == "gen" else kind, n, perm)
    return spec, n, conn, nn


def parse_list(csv: str, valid, what: str):
    out = []
    for item in csv.split(","):
        if item in ("spin", "spin-vec"):
            raise UsageError(f"method '{item}' has no GPU counterpart (per-row spin locks); use seq")
        if item not in valid:
            raise UsageError(f"unknown {what} '{item}' (valid: {', '.join(valid)})")
        if item not in out:
            out.append(item)
    if not out:
        raise UsageError(f"no {what}s given")
    return out


def write_matrix_market(row_ptr, cols, values, os) -> None:
    """write_matrix_market (formats.hpp:366-379): 1-based coordinates, %.17g values."""
    n = len(row_ptr) - 1
    os.write("%%MatrixMarket matrix coordinate real general\n")
    os.write(f"{n} {n} {len(values)}\n")
    rows = np.repeat(np.arange(1, n + 1), np.diff(row_ptr))
    for r, c, v in zip(rows, cols + 1, values):
        os.write(f"{r} {c} {v:.17g}\n")


def write_raw_csv(cases, os) -> None:
    os.write("suite,mesh,n,p,d,dofs,nnz,method,format,threads,run,micros\n")
    for c in cases:
        for i, t in enumerate(c["t_micros"]):
            os.write(f"{_prefix(c)},{i + 1},{t:.3f}\n")


def write_summary_csv(cases, os) -> None:
    os.write("suite,mesh,n,p,d,dofs,nnz,method,format,threads,t_avg,t_min,c,gamma,values_mb\n")
    for c in cases:
        os.write(f"{_prefix(c)},{c['t_avg']:.3f},{c['t_min']:.3f},{c['c']:.4f},{c['gamma']:.6f},"
                 f"{c['values_mb']:.6f}\n")


def print_summary(cases, os) -> None:
    os.write("%-10s %3s %3s %10s %10s %-10s %-5s %3s %12s %12s %7s %7s\n" %
             ("mesh", "p", "d", "dofs", "nnz", "method", "fmt", "thr", "t_avg[us]", "t_min[us]", "c", "gamma"))
    for c in cases:
        os.write("%-10s %3d %3d %10d %10d %-10s %-5s %3d %12.2f %12.2f %7.3f %7.4f\n" %
                 (c["mesh"][:10], c["p"], c["d"], c["dofs"], c["nnz"], c["method"], c["format"], c["threads"],
                  c["t_avg"], c["t_min"], c["c"], c["gamma"]))


def _prefix(c) -> str:
    return (f"{c['suite']},{c['mesh']},{c['n']},{c['p']},{c['d']},{c['dofs']},{c['nnz']},{c['method']},"
            f"{c['format']},{c['threads']}")


# ---------------------------------------------------------------------------- GPU commands

def _plan(conn, nn, d):
    from .assembly import Plan
    return Plan(M.element_dofs(conn, d), nn * d, dofs_per_node=d)


def _time_assembly(plan, K, values, strategy, runs):
    """time_assembly (bench.hpp:98-113): untimed reset + one warm-up, then `runs` timed
    assemblies on reset values (CUDA events, microseconds). The deterministic segmented
    reductions write every slot, so they run in overwrite mode (== reset + assemble, same bits);
    atomics add into the reset array."""
    import torch
    acc = strategy == "atomic"
    values.zero_()
    plan.assemble(K, values, strategy=strategy, accumulate=acc)
    out = []
    for _ in range(runs):
        values.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.assemble(K, values, strategy=strategy, accumulate=acc)
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return out


def cmd_assemble(a) -> int:
    import torch
    from .assembly import fill_seeded_k
    label, n, conn, nn = parse_mesh(a.mesh)
    plan = _plan(conn, nn, a.d)
    strategy = METHODS[a.method]
    if strategy == "colour":
        plan.set_colouring(plan.greedy_colouring()[0])
    K = fill_seeded_k(conn.shape[0], conn.shape[1] * a.d, a.seed)
    values = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
    t = _time_assembly(plan, K, values, strategy, 1)[0]
    print(f"mesh {label}: {plan.n_rows} dofs, {plan.nnz} nnz, {plan.n_runs} runs; method {a.method}, "
          f"format {a.format}: {t:.2f} us")
    if a.dump:
        # fea_main.cpp:239-253: the dump is ones_supplier + assemble_sequential into CSR
        ones = torch.ones_like(K)
        dumped = plan.assemble(ones, strategy="sorted")
        rp, cs = plan.csr()
        with open(a.dump, "w") as f:
            write_matrix_market(rp, cs, dumped.cpu().numpy(), f)
        print(f"wrote {a.dump}")
    return EXIT_OK


def cmd_bench(a) -> int:
    import torch
    from .assembly import fill_seeded_k
    methods = parse_list(a.methods, list(METHODS), "method")
    formats = parse_list(a.formats, list(FORMATS), "format")
    label, n, conn, nn = parse_mesh(a.mesh)
    plan = _plan(conn, nn, a.d)
    if "colour-vec" in methods:
        plan.set_colouring(plan.greedy_colouring()[0])
    K = fill_seeded_k(conn.shape[0], conn.shape[1] * a.d, a.seed)
    values = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
    gamma = (2 * plan.n_runs + 2) / plan.nnz if plan.nnz else 0.0  # storage_factor, bench.cpp:100-113
    cases, t_seq = [], {}
    for fmt in formats:  # one values kernel serves both formats; timed per format like the reference
        for meth in methods:
            ts = _time_assembly(plan, K, values, METHODS[meth], a.runs)
            c = dict(suite="single", mesh=label, n=n, p=1, d=a.d, dofs=plan.n_rows, nnz=plan.nnz, method=meth,
                     format=fmt, threads=a.threads, t_micros=ts, t_avg=float(np.mean(ts)), t_min=float(np.min(ts)),
                     gamma=gamma, values_mb=8.0 * plan.nnz / 1e6)
            if meth == "seq":
                t_seq[fmt] = c["t_avg"]
            cases.append(c)
    for c in cases:  # speed factor vs seq of the same format (bench.cpp:93-98)
        c["c"] = t_seq.get(c["format"], c["t_avg"]) / c["t_avg"]
    print_summary(cases, sys.stdout)
    if a.out:
        with open(a.out + ".raw.csv", "w") as f:
            write_raw_csv(cases, f)
        with open(a.out + ".summary.csv", "w") as f:
            write_summary_csv(cases, f)
    return EXIT_OK


@dataclass
class VerifyResult:
    """fea::VerifyResult (verify.hpp:38-45)."""
    ok: bool = True
    dofs: int = 0
    nnz: int = 0
    expected_total: float = 0.0
    checked: list = field(default_factory=list)
    failures: list = field(default_factory=list)


def _compare_values(combo, got, want, expected_total, out: VerifyResult) -> None:
    """compare_values (verify.cpp:31-54): first differing slot by bit pattern, then the exact
    total; messages in the reference's wording (std::to_string -> %f)."""
    if got.size != want.size:
        out.failures.append(f"{combo}: values length mismatch")
        return
    diff = np.flatnonzero(got.view(np.int64) != want.view(np.int64))
    if diff.size:
        i = int(diff[0])
        out.failures.append(f"{combo}: values[{i}] = {got[i]:f}, sequential has {want[i]:f}")
        return
    total = float(np.sum(got))
    if total != expected_total:
        out.failures.append(f"{combo}: total {total:f} != expected {expected_total:f}")


def verify_methods(conn, n_nodes: int, d: int, tamper=None) -> VerifyResult:
    """verify_methods (verify.cpp:70-156) on the GPU: ones element matrices, every GPU method on
    both formats, bitwise equal to seq/csr and totals exactly E*m^2. `tamper(combo, values)`
    is the reference's test hook (VerifyOptions::tamper, verify.hpp:31-36), called with each
    combination's host values right after its assembly. The spin methods have no GPU
    counterpart, so 6 combinations are checked (the reference checks 10)."""
    import torch
    plan = _plan(conn, n_nodes, d)
    plan.set_colouring(plan.greedy_colouring()[0])
    E, m = conn.shape[0], conn.shape[1] * d
    K = torch.ones((E, m, m), dtype=torch.float64, device=f"cuda:{plan.device}")
    out = VerifyResult(dofs=plan.n_rows, nnz=plan.nnz, expected_total=float(E) * m * m)
    ref = plan.assemble(K, strategy="sorted").cpu().numpy()
    total = float(np.sum(ref))
    if total != out.expected_total:
        out.failures.append(f"seq/csr: total {total:f} != expected {out.expected_total:f}")
    out.checked.append("seq/csr")
    for meth in METHODS:
        for fmt in FORMATS:
            combo = f"{meth}/{fmt}"
            if combo == "seq/csr":
                continue
            got = plan.assemble(K, strategy=METHODS[meth]).cpu().numpy()
            if tamper is not None:
                tamper(combo, got)
            _compare_values(combo, got, ref, out.expected_total, out)
            out.checked.append(combo)
    out.ok = not out.failures
    return out


def parse_tamper(spec):
    """--tamper COMBO:INDEX[:DELTA] -> a tamper hook adding DELTA (default 1.0) to values[INDEX]
    of that combination (the reference's test hook exposed on the command line)."""
    if not spec:
        return None
    parts = spec.split(":")
    if len(parts) not in (2, 3) or parts[0] not in [f"{m}/{f}" for m in METHODS for f in FORMATS]:
        raise UsageError(f"--tamper '{spec}': expected METHOD/FORMAT:INDEX[:DELTA]")
    combo, idx = parts[0], int(parts[1])
    delta = float(parts[2]) if len(parts) == 3 else 1.0

    def hook(c, values):
        if c == combo:
            values[idx] += delta
    return hook


def cmd_verify(a) -> int:
    """fea verify (fea_main.cpp:305-318): exit 0 when every combination matches, 2 otherwise."""
    label, n, conn, nn = parse_mesh(a.mesh)
    res = verify_methods(conn, nn, a.d, tamper=parse_tamper(a.tamper))
    print(f"dofs: {res.dofs}, nnz: {res.nnz}, combinations: {len(res.checked)}, threads: {a.threads}")
    if res.ok:
        print("verify: OK (all methods bitwise identical, totals exact)")
        return EXIT_OK
    for f in res.failures:
        print(f"verify: FAIL {f}")
    return EXIT_VERIFY_FAILED


def cmd_colour(a) -> int:
    from .assembly import Plan
    label, n, conn, nn = parse_mesh(a.mesh)
    plan = Plan(M.element_dofs(conn, 1), nn)
    col, nc = plan.jp_colouring(seed=a.seed) if a.jp else plan.greedy_colouring()
    print(f"mesh {label}: {len(col)} elements, {nc} colours")
    for c in range(nc):  # colour_distribution, colouring.cpp:77-89
        print(f"  colour {c}: {np.count_nonzero(col == c) / max(len(col), 1):.4f}")
    if a.out:
        with open(a.out, "w") as f:  # write_colouring_csv, colouring.cpp:121-127
            f.write("element,colour\n")
            for e, c in enumerate(col):
                f.write(f"{e},{c}\n")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="fea-gpu", description="Parallel FE assembly into CSR/CRAC on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("assemble", help="Run one assembly and report timing")
    s.add_argument("--mesh", default="gen:8")
    s.add_argument("--p", type=int, default=1)
    s.add_argument("--d", type=int, default=1)
    s.add_argument("--method", default="seq", choices=list(METHODS))
    s.add_argument("--format", default="csr", choices=list(FORMATS))
    s.add_argument("--threads", type=int, default=1)
    s.add_argument("--seed", type=int, default=M.SEED_K)
    s.add_argument("--dump", default=None, help="write the result in Matrix Market format")
    s = sub.add_parser("bench", help="Time methods x formats, write raw+summary CSV")
    s.add_argument("--suite", default="single", choices=["single"])
    s.add_argument("--mesh", default="gen:256")
    s.add_argument("--p", type=int, default=1)
    s.add_argument("--d", type=int, default=1)
    s.add_argument("--methods", default="seq,atomic,colour-vec")
    s.add_argument("--formats", default="csr,crac")
    s.add_argument("--runs", type=int, default=30)
    s.add_argument("--threads", type=int, default=1)
    s.add_argument("--seed", type=int, default=M.SEED_K)
    s.add_argument("--out", default=None, help="output prefix: <out>.raw.csv, <out>.summary.csv")
    s = sub.add_parser("verify", help="All methods x formats bitwise equal with ones matrices")
    s.add_argument("--mesh", default="gen:48")
    s.add_argument("--p", type=int, default=1)
    s.add_argument("--d", type=int, default=1)
    s.add_argument("--threads", type=int, default=1)
    s.add_argument("--tamper", default=None,
                   help="test hook: METHOD/FORMAT:INDEX[:DELTA] corrupts one slot of that combination")
    s = sub.add_parser("colour", help="Greedy element colouring report")
    s.add_argument("--mesh", default="gen:8")
    s.add_argument("--p", type=int, default=1)
    s.add_argument("--out", default=None, help="CSV dump path (element,colour)")
    s.add_argument("--jp", action="store_true", help="Jones-Plassmann colouring on the GPU instead of greedy")
    s.add_argument("--seed", type=int, default=1)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        if getattr(a, "p", 1) != 1:
            raise UsageError("p > 1 (hierarchical DOF numbering) is out of scope; use the 3D Q2 mesh hex27:N")
        if getattr(a, "d", 1) < 1 or getattr(a, "runs", 1) < 1:
            raise UsageError("d and runs must be >= 1")
        return {"assemble": cmd_assemble, "bench": cmd_bench, "verify": cmd_verify, "colour": cmd_colour}[a.cmd](a)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001 — the reference maps every other failure to 3
        print(f"error: {e}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
