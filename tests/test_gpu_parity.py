"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Patterns and CRAC arrays: bit-exact int64 arrays (build_pattern pattern.cpp:24-108,
build_crac_arrays formats.cpp:21-41). Values: FEA_DET_SORTED bit-exact vs
assemble_sequential (assembly.hpp:112-118); FEA_DET_COLOUR bit-exact vs
assemble_coloured_vectorized (assembly.hpp:175-195) under the same greedy colouring;
FEA_ATOMIC within |a-b| <= 1e-12*max(|a|,|b|,1) (test_assembly.cpp:236).
"""
import numpy as np
import pytest

from paper_2012_00585_b200 import meshgen as M

pytestmark = pytest.mark.gpu

TOL = 1e-12  # reference tolerance form, test_assembly.cpp:236 / acceptance.cpp:281

CASES = [
    ("quad4", 6, 1, None),
    ("quad4", 4, 5, None),          # d >= 5: the generic gathers and k_scatter atomics
    ("quad4", 3, 8, "nodes"),       # the paper's d-benchmark goes up to 8
    ("hex8", 2, 5, "elements"),
    ("quad4", 5, 4, "nodes"),
    ("hex8", 3, 3, "elements"),
    ("hex8", 4, 2, None),
    ("tet4", 4, 1, "nodes"),
    ("tet4", 3, 3, None),
    ("hex27", 2, 3, None),
    ("hex27", 3, 1, "elements"),
]


def close(a, b, tol=TOL):
    return np.all(np.abs(a - b) <= tol * np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0))


def problem(mesh, n, d, perm):
    conn, nn = M.make_mesh(mesh, n, perm)
    return conn, nn, M.element_dofs(conn, d), nn * d


@pytest.mark.parametrize("mesh,n,d,perm", CASES)
def test_pattern_bit_exact(gpu, orc, mesh, n, d, perm):
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    P = orc.Pattern.build(conn, nn, d)
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        assert plan.dofs_per_node == d
        assert (plan.n_rows, plan.nnz, plan.n_runs) == (P.n_rows, P.nnz, P.n_runs)
        rp, cs = plan.csr()
        orp, ocs = P.arrays()
        assert np.array_equal(rp, orp) and np.array_equal(cs, ocs)
        cp, ca = plan.crac()
        ocp, oca = P.crac()
        assert np.array_equal(cp, ocp) and np.array_equal(ca, oca)
    if perm is None:
        assert P.nnz == M.closed_form_nnz(mesh, n, d)


@pytest.mark.parametrize("mesh,n,d,perm", CASES)
def test_seeded_k_matches_oracle(gpu, orc, mesh, n, d, perm):
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    K = gpu.fill_seeded_k(conn.shape[0], ed.shape[1], 42).cpu().numpy()
    assert K.tobytes() == orc.fill_k(42, conn.shape[0], ed.shape[1]).tobytes()
    assert np.array_equal(K, np.swapaxes(K, 1, 2))


@pytest.mark.parametrize("mesh,n,d,perm", CASES)
def test_values_all_strategies(gpu, orc, mesh, n, d, perm):
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(42, conn.shape[0], ed.shape[1])
    want_seq = P.assemble_sequential(ed, Kh)
    col, nc = orc.greedy_colouring(conn, nn)
    want_col = P.assemble_coloured(ed, Kh, col)
    K = torch.from_numpy(Kh).cuda()
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        got = plan.assemble(K, strategy="sorted").cpu().numpy()
        assert got.tobytes() == want_seq.tobytes()
        gcol, gnc = plan.greedy_colouring()
        assert np.array_equal(gcol, col) and gnc == nc
        plan.set_colouring(gcol)
        got_c = plan.assemble(K, strategy="colour").cpu().numpy()
        assert got_c.tobytes() == want_col.tobytes()
        got_p = plan.assemble(K, strategy="colour_passes").cpu().numpy()
        assert got_p.tobytes() == want_col.tobytes()
        got_a = plan.assemble(K, strategy="atomic").cpu().numpy()
        assert close(got_a, want_seq)


@pytest.mark.parametrize("mesh,n,d,perm", CASES[:5])
def test_ones_bitwise_and_conservation(gpu, orc, mesh, n, d, perm):
    """acceptance.cpp:180-199 / verify.cpp:85-100: with ones K every route is bitwise equal
    to sequential and the total is exactly E*m^2."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, d)
    want = P.assemble_sequential(ed, np.ones((E, m, m)))
    K = torch.ones((E, m, m), dtype=torch.float64, device="cuda")
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        col, _ = plan.greedy_colouring()
        plan.set_colouring(col)
        for s in ("sorted", "atomic", "colour", "colour_passes"):
            got = plan.assemble(K, strategy=s).cpu().numpy()
            assert got.tobytes() == want.tobytes(), s
            assert got.sum() == E * m * m


@pytest.mark.parametrize("strategy", ["sorted", "atomic", "colour", "colour_passes"])
def test_accumulate_twice_doubles(gpu, orc, strategy):
    """test_assembly.cpp:89-99: assembling twice without reset doubles every value."""
    import torch
    conn, nn, ed, n_rows = problem("quad4", 3, 2, None)
    E, m = ed.shape
    K = torch.ones((E, m, m), dtype=torch.float64, device="cuda")
    with gpu.Plan(ed, n_rows, dofs_per_node=2) as plan:
        plan.set_colouring(plan.greedy_colouring()[0])
        v = plan.assemble(K, strategy=strategy)
        once = v.clone()
        plan.assemble(K, v, strategy=strategy, accumulate=True)
        assert torch.equal(v, 2 * once)


@pytest.mark.parametrize("mesh,n,d,perm", [("hex8", 3, 3, "elements"), ("tet4", 4, 1, "nodes"),
                                            ("quad4", 6, 1, None)])
def test_accumulate_is_left_fold_from_existing(gpu, orc, mesh, n, d, perm):
    """FEA_ACCUMULATE on the sorted route continues the fold from the slot's value,
    exactly like assemble_sequential on a non-reset target."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(5, conn.shape[0], ed.shape[1])
    start = orc.fill_k(9, 1, int(np.ceil(np.sqrt(P.nnz))))[0].reshape(-1)[: P.nnz].copy()
    want = P.assemble_sequential(ed, Kh, start.copy())
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        v = torch.from_numpy(start.copy()).cuda()
        plan.assemble(torch.from_numpy(Kh).cuda(), v, strategy="sorted", accumulate=True)
        assert v.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("where", ["host", "device"])
@pytest.mark.parametrize("fmt", ["csr", "crac"])
def test_external_pattern_superset(gpu, orc, fmt, where):
    """A caller's pattern with extra entries (random_pattern-style superset): slots resolved
    by the device CSR search / CRAC Listing-1 search; values bit-exact vs sequential."""
    import torch
    conn, nn, ed, n_rows = problem("quad4", 4, 2, "nodes")
    P = orc.Pattern.build(conn, nn, 2)
    rp, cs = P.arrays()
    rng = np.random.default_rng(3)
    rows = []
    for r in range(n_rows):
        extra = rng.choice(n_rows, size=3, replace=False)
        rows.append(np.unique(np.concatenate([cs[rp[r]:rp[r + 1]], extra])))
    srp = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    scs = np.concatenate(rows).astype(np.int64)
    S = orc.Pattern.from_arrays(srp, scs)
    Kh = orc.fill_k(1, conn.shape[0], ed.shape[1])
    want = S.assemble_sequential(ed, Kh)
    put = (lambda a: torch.from_numpy(a).cuda()) if where == "device" else (lambda a: a)
    if fmt == "csr":
        plan = gpu.Plan.with_pattern(ed, n_rows, put(srp), put(scs), "csr")
    else:
        cp, ca = S.crac()
        plan = gpu.Plan.with_pattern(ed, n_rows, put(cp), put(ca), "crac")
    with plan:
        assert plan.nnz == S.nnz and plan.missing_entry() is None
        prp, pcs = plan.csr()  # the plan's view of the caller's pattern (CRAC: expanded on the device)
        assert np.array_equal(prp, srp) and np.array_equal(pcs, scs)
        got = plan.assemble(torch.from_numpy(Kh).cuda(), strategy="sorted").cpu().numpy()
        assert got.tobytes() == want.tobytes()
        got_a = plan.assemble(torch.from_numpy(Kh).cuda(), strategy="atomic").cpu().numpy()
        assert close(got_a, want)


def test_external_pattern_malformed_is_invalid(gpu, orc):
    """Malformed caller patterns are refused with FEA_ERR_INVALID (ValueError) before any
    indexing: row_ptr[0] != 0, decreasing row_ptr, odd CRAC row pointers, CRAC value positions
    that do not follow the runs, columns outside the matrix."""
    conn, nn, ed, n_rows = problem("quad4", 3, 1, None)
    P = orc.Pattern.build(conn, nn, 1)
    rp, cs = P.arrays()
    cp, ca = P.crac()
    bad = []
    r = rp.copy(); r[0] = 1; bad.append((r, cs, "csr"))
    r = rp.copy(); r[3] = r[4] + 1; bad.append((r, cs, "csr"))
    c = cs.copy(); c[5] = n_rows + 7; bad.append((rp, c, "csr"))
    r = cp.copy(); r[2] += 1; bad.append((r, ca, "crac"))
    a = ca.copy(); a[3] = a[5] + 2; bad.append((cp, a, "crac"))
    a = ca.copy(); a[-1] = a[-3]; bad.append((cp, a, "crac"))
    a = ca.copy(); a[-4] = n_rows; bad.append((cp, a, "crac"))
    c = cs.copy(); c[rp[2]], c[rp[2] + 1] = c[rp[2] + 1], c[rp[2]]; bad.append((rp, c, "csr"))  # not ascending
    c = cs.copy(); c[0] = -1; bad.append((rp, c, "csr"))
    r = rp.copy(); r[-1] = -5; bad.append((r, cs, "csr"))
    for r, c, fmt in bad:
        with pytest.raises(ValueError):
            gpu.Plan.with_pattern(ed, n_rows, r, c, fmt)
    with gpu.Plan.with_pattern(ed, n_rows, cp, ca, "crac") as plan:  # the well-formed one
        assert plan.nnz == P.nnz


def test_missing_entry_is_assembly_error(gpu, orc):
    """test_assembly.cpp:122-141: pattern of the first element only, all four assembled."""
    import torch
    conn, nn = M.quad4_structured(2)
    ed = M.element_dofs(conn, 1)
    P = orc.Pattern.build(conn[:1], nn, 1)
    rp, cs = P.arrays()
    with gpu.Plan.with_pattern(ed, nn, rp, cs, "csr") as plan:
        miss = plan.missing_entry()
        assert miss is not None and miss[0] == 1
        with pytest.raises(gpu.AssemblyError, match="element 1"):
            plan.assemble(torch.ones((4, 4, 4), dtype=torch.float64, device="cuda"))
    with pytest.raises(orc.MissingEntry) as ei:
        P.assemble_sequential(ed, np.ones((4, 4, 4)))
    assert ei.value.args[0] == miss


def test_invalid_colouring_rejected(gpu):
    """test_assembly.cpp:329-348: a single-colour colouring of a 2x2 mesh conflicts."""
    conn, nn = M.quad4_structured(2)
    with gpu.Plan(M.element_dofs(conn, 1), nn) as plan:
        with pytest.raises(gpu.AssemblyError, match="share dof"):
            plan.set_colouring(np.zeros(4, np.int32))


@pytest.mark.parametrize("k_compact", [False, True])
@pytest.mark.parametrize("mesh,n,d,perm", [("hex8", 4, 3, "elements"), ("tet4", 4, 1, "nodes")])
def test_row_partition_blocks_concatenate(gpu, orc, k_compact, mesh, n, d, perm):
    """Row-partitioned plans: each owned block's CSR/CRAC/values equal the matching slice
    of the whole-matrix result. tet4 d=1 with permuted node ids runs the
    traversal-ordered d = 1 gather on each block."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    P = orc.Pattern.build(conn, nn, d)
    rp, cs = P.arrays()
    Kh = orc.fill_k(42, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    cuts = [0, d * 40, d * 41, d * 90, n_rows]
    for rb, re in zip(cuts[:-1], cuts[1:]):
        with gpu.Plan(ed, n_rows, dofs_per_node=d, row_range=(rb, re), k_compact=k_compact) as plan:
            prp, pcs = plan.csr()
            assert np.array_equal(prp, rp[rb:re + 1] - rp[rb])
            assert np.array_equal(pcs, cs[rp[rb]:rp[re]])
            ids = plan.elements()
            Kp = torch.from_numpy(Kh[ids] if k_compact else Kh).cuda()
            for s in ("sorted", "atomic"):
                got = plan.assemble(Kp, strategy=s).cpu().numpy()
                sl = want[rp[rb]:rp[re]]
                if s == "sorted":
                    assert got.tobytes() == sl.tobytes()
                else:
                    assert close(got, sl)


def test_host_end_to_end(gpu, orc):
    conn, nn, ed, n_rows = problem("hex8", 3, 3, "elements")
    P = orc.Pattern.build(conn, nn, 3)
    Kh = orc.fill_k(42, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    with gpu.Plan(ed, n_rows, dofs_per_node=3) as plan:
        got = plan.assemble_host(Kh, strategy="sorted")
        assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("mesh,n,d,perm", [("hex8", 6, 3, None), ("hex8", 5, 3, "elements"),
                                            ("tet4", 5, 1, "nodes"), ("quad4", 16, 1, None),
                                            ("hex27", 3, 3, None), ("hex8", 5, 1, None), ("quad4", 9, 5, None)])
@pytest.mark.parametrize("windows", [1, 5, 13])
def test_host_windowed_pipeline(gpu, orc, mesh, n, d, perm, windows):
    """fea_assemble_host in traversal windows (K chunks uploaded as windows need them, each
    window's values downloaded as it completes): bit-exact vs assemble_sequential /
    assemble_coloured_vectorized, overwrite and accumulate; atomic within 1e-12."""
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(7, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    col, _ = orc.greedy_colouring(conn, nn)
    want_c = P.assemble_coloured(ed, Kh, col)
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        plan.set_host_windows(windows)
        plan.set_colouring(plan.greedy_colouring()[0])
        for rep in range(2):  # second call reuses staging, streams and window tables
            assert plan.assemble_host(Kh, strategy="sorted").tobytes() == want.tobytes()
        assert plan.assemble_host(Kh, strategy="colour").tobytes() == want_c.tobytes()
        start = np.full(P.nnz, 0.25)
        got = plan.assemble_host(Kh, start.copy(), strategy="sorted", accumulate=True)
        assert got.tobytes() == P.assemble_sequential(ed, Kh, start.copy()).tobytes()
        assert close(plan.assemble_host(Kh, strategy="atomic"), want)


def test_empty_and_degenerate(gpu):
    """test_formats.cpp:111-139: empty pattern / empty rows."""
    import torch
    ed = np.zeros((0, 4), np.int64)
    with gpu.Plan(ed, 0) as plan:
        assert (plan.n_rows, plan.nnz, plan.n_runs) == (0, 0, 0)
        rp, ca = plan.crac()
        assert list(rp) == [0] and list(ca) == [0, 0]
    # rows with no element (isolated DOFs 4..7)
    conn, nn = M.quad4_structured(1)
    with gpu.Plan(M.element_dofs(conn, 1), 8) as plan:
        rp, cs = plan.csr()
        assert list(rp[4:]) == [16, 16, 16, 16, 16]
        v = plan.assemble(torch.ones((1, 4, 4), dtype=torch.float64, device="cuda"))
        assert torch.all(v == 1.0)


GOLDEN = ["quad4_n6_d1", "quad4_n5_d2_nodeperm", "hex8_n3_d3_elemperm", "tet4_n3_d1_nodeperm",
          "hex27_n2_d3", "hex8_n4_d1", "refdofmap_n4_p3_d2"]


@pytest.mark.parametrize("name", GOLDEN)
def test_gpu_matches_reference_fixtures(gpu, orc, name):
    """The CUDA path against arrays produced by the unmodified reference library
    (tests/golden/make_golden.py): patterns/CRAC bit-exact, sequential and colour-vec values
    bit-exact, atomics within 1e-12, ones-K exact."""
    import torch
    from tests.test_oracle import gold_case
    g, conn, nn, d = gold_case(name)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        rp, cs = plan.csr()
        assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(cs, g["cols"])
        cp, ca = plan.crac()
        assert np.array_equal(cp, g["crac_ptr"]) and np.array_equal(ca, g["col_align"])
        col, nc = plan.greedy_colouring()
        assert np.array_equal(col, g["colour_of"]) and nc == int(g["n_colours"])
        plan.set_colouring(col)
        K = gpu.fill_seeded_k(E, m, 42)
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == g["values_seq"].tobytes()
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == g["values_colour"].tobytes()
        assert plan.assemble(K, strategy="colour_passes").cpu().numpy().tobytes() == g["values_colour"].tobytes()
        assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), g["values_seq"])
        ones = torch.ones((E, m, m), dtype=torch.float64, device="cuda")
        for s in ("sorted", "atomic", "colour"):
            assert plan.assemble(ones, strategy=s).cpu().numpy().tobytes() == g["values_ones"].tobytes()


def test_host_batch_pipeline(gpu, orc):
    """fea_assemble_host_batch: several steps with different K, each bit-exact vs sequential."""
    import torch
    conn, nn, ed, n_rows = problem("hex8", 3, 3, "elements")
    P = orc.Pattern.build(conn, nn, 3)
    Ks = [orc.fill_k(s, conn.shape[0], ed.shape[1]) for s in (1, 2, 3, 4, 5)]
    vals = [np.zeros(P.nnz) for _ in Ks]
    with gpu.Plan(ed, n_rows, dofs_per_node=3) as plan:
        for strategy in ("sorted", "atomic"):
            plan.assemble_host_batch(Ks, vals, strategy=strategy)
            for K, v in zip(Ks, vals):
                want = P.assemble_sequential(ed, K)
                if strategy == "sorted":
                    assert v.tobytes() == want.tobytes()
                else:
                    assert close(v, want)
        # accumulate: values are uploaded, added to, downloaded
        start = [np.full(P.nnz, 0.5) for _ in Ks[:2]]
        plan.assemble_host_batch(Ks[:2], start, strategy="sorted", accumulate=True)
        for K, v in zip(Ks[:2], start):
            assert v.tobytes() == P.assemble_sequential(ed, K, np.full(P.nnz, 0.5)).tobytes()


@pytest.mark.parametrize("mesh,n,d,perm", CASES)
def test_spmv_csr_crac_nodes(gpu, orc, mesh, n, d, perm):
    """y = A x through the CSR, CRAC and node-block kernels against a host CSR product
    (different summation order than the host: |y - y_ref| <= 1e-12 * (|A| |x|) per row)."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        K = gpu.fill_seeded_k(conn.shape[0], ed.shape[1], 3)
        vals = plan.assemble(K, strategy="sorted")
        rp, cs = plan.csr()
        cp, ca = plan.crac()
        x = np.random.default_rng(1).uniform(-1, 1, n_rows)
        v = vals.cpu().numpy()
        rows = np.repeat(np.arange(n_rows), np.diff(rp))
        want = np.bincount(rows, weights=v * x[cs], minlength=n_rows)
        scale = np.bincount(rows, weights=np.abs(v * x[cs]), minlength=n_rows)
        xd = torch.from_numpy(x).cuda()
        for got in (gpu.spmv_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(cs).cuda(), vals, xd),
                    gpu.spmv_crac(torch.from_numpy(cp).cuda(), torch.from_numpy(ca).cuda(), vals, xd),
                    *((plan.spmv(vals, xd),) if d <= 4 else ())):  # node-block kernel: d <= 4
            g = got.cpu().numpy()
            assert np.all(np.abs(g - want) <= 1e-12 * np.maximum(scale, 1e-300) + 1e-300)


@pytest.mark.parametrize("mesh,n,d,perm", CASES)
def test_fused_supplier_bitwise(gpu, mesh, n, d, perm):
    """fea_assemble_seeded (K generated inside the gather) == fea_assemble on a materialized seeded K."""
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        K = gpu.fill_seeded_k(conn.shape[0], ed.shape[1], 11)
        want = plan.assemble(K, strategy="sorted")
        got = plan.assemble_seeded(11, strategy="sorted")
        assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
        plan.set_colouring(plan.greedy_colouring()[0])
        assert plan.assemble_seeded(11, strategy="colour").cpu().numpy().tobytes() == \
            plan.assemble(K, strategy="colour").cpu().numpy().tobytes()


def test_fused_supplier_partitioned_compact(gpu):
    conn, nn, ed, n_rows = problem("hex8", 4, 3, "elements")
    with gpu.Plan(ed, n_rows, dofs_per_node=3) as full:
        want = full.assemble_seeded(5).cpu().numpy()
        rp, _ = full.csr()
    rb, re = 3 * 40, 3 * 90
    with gpu.Plan(ed, n_rows, dofs_per_node=3, row_range=(rb, re), k_compact=True) as plan:
        got = plan.assemble_seeded(5).cpu().numpy()
        assert got.tobytes() == want[rp[rb]:rp[re]].tobytes()


@pytest.mark.parametrize("mesh,n,d,perm", CASES[:6])
def test_jones_plassmann_colouring(gpu, orc, mesh, n, d, perm):
    """GPU Jones-Plassmann colouring is valid (no two same-colour elements share a node) and the
    colour routes are bit-identical to the reference's coloured assembly under it."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        col, nc = plan.jp_colouring(seed=3)
        assert col.min() == 0 and col.max() == nc - 1
        for c in range(nc):
            nodes = conn[col == c].reshape(-1)
            assert len(np.unique(nodes)) == len(nodes)
        plan.set_colouring(col)
        P = orc.Pattern.build(conn, nn, d)
        Kh = orc.fill_k(8, conn.shape[0], ed.shape[1])
        want = P.assemble_coloured(ed, Kh, col)
        K = torch.from_numpy(Kh).cuda()
        for s in ("colour", "colour_passes"):
            assert plan.assemble(K, strategy=s).cpu().numpy().tobytes() == want.tobytes()


def test_colouring_of_partitioned_plan_checks_owned_rows_only(gpu, orc):
    import torch
    conn, nn, ed, n_rows = problem("hex8", 4, 3, "elements")
    rb, re = 3 * 40, 3 * 90
    with gpu.Plan(ed, n_rows, dofs_per_node=3, row_range=(rb, re)) as plan:
        col, nc = plan.jp_colouring(seed=1)
        plan.set_colouring(col)
        P = orc.Pattern.build(conn, nn, 3)
        rp, _ = P.arrays()
        ids = plan.elements()
        Kh = orc.fill_k(2, conn.shape[0], ed.shape[1])
        full_col = np.full(conn.shape[0], 0, np.int32)
        # the reference colour-vec over the kept elements with this colouring, restricted to owned rows
        Pk = orc.Pattern.build(conn[ids], nn, 3)
        want = Pk.assemble_coloured(ed[ids], Kh[ids], col)
        rpk, _ = Pk.arrays()
        got = plan.assemble(torch.from_numpy(Kh).cuda(), strategy="colour").cpu().numpy()
        assert got.tobytes() == want[rpk[rb]:rpk[re]].tobytes()
        del full_col, rp


DEGENERATE = [("quad4", 5, 1, None), ("quad4", 4, 2, "nodes"), ("hex8", 3, 3, "elements"),
              ("hex8", 3, 1, None), ("tet4", 3, 1, "nodes"), ("tet4", 2, 3, None), ("hex27", 2, 1, None)]


@pytest.mark.parametrize("mesh,n,d,perm", DEGENERATE)
def test_degenerate_elements_all_strategies(gpu, orc, mesh, n, d, perm):
    """Elements listing a node twice (collapsed quads / wedges): one element row block then
    hits the same slot from two columns, folded in column order like scatter_element
    (assembly.hpp:77-92); sorted / colour / colour passes stay bit-exact."""
    import torch
    conn, nn = M.make_mesh(mesh, n, perm)
    conn = M.collapse_elements(conn, np.random.default_rng(n * 10 + d))
    ed = M.element_dofs(conn, d)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(3, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    col, _ = orc.greedy_colouring(conn, nn)
    want_col = P.assemble_coloured(ed, Kh, col)
    K = torch.from_numpy(Kh).cuda()
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        assert plan.nnz == P.nnz
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        assert plan.assemble_seeded(3, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        plan.set_colouring(col)
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == want_col.tobytes()
        assert plan.assemble(K, strategy="colour_passes").cpu().numpy().tobytes() == want_col.tobytes()
        assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)


def _hub_mesh(kind):
    """Quads around a hub node: 'wide' - 200 quads, each with 3 nodes of its own (the hub has 800
    candidate nodes and a row of 601 columns: block-per-node pattern kernel, 2-byte positions);
    'dense' - 140 quads drawn from a ring of 40 nodes (560 candidates, a row of 41 columns:
    block-per-node kernel with byte positions)."""
    if kind == "wide":
        conn = np.array([[0, 3 * i + 1, 3 * i + 2, 3 * i + 3] for i in range(200)], np.int64)
        return conn, 601
    ring = 40
    conn = np.array([[0, 1 + i % ring, 1 + (i * 7 + 3) % ring, 1 + (i * 11 + 5) % ring] for i in range(140)], np.int64)
    return conn, ring + 1


@pytest.mark.parametrize("env", [{}, {"FEA_PLAN_NO_FUSED": "1"}])
@pytest.mark.parametrize("kind,d", [("wide", 1), ("wide", 2), ("dense", 1), ("dense", 3)])
def test_high_valence_hub(gpu, orc, kind, d, env, monkeypatch):
    """A node with more than 512 candidate column nodes takes the block-per-node pattern kernel
    (k_node_pattern_big), and the fused symbolic pass hands over to the separate count / fill /
    slot-map passes; pattern, CRAC arrays and every strategy against the oracle."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    conn, nn = _hub_mesh(kind)
    ed = M.element_dofs(conn, d)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(21, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    col, _ = orc.greedy_colouring(conn, nn)
    want_col = P.assemble_coloured(ed, Kh, col)
    K = torch.from_numpy(Kh).cuda()
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        rp, cs = plan.csr()
        orp, ocs = P.arrays()
        assert np.array_equal(rp, orp) and np.array_equal(cs, ocs)
        crp, cal = plan.crac()
        ocrp, ocal = P.crac()
        assert np.array_equal(crp, ocrp) and np.array_equal(cal, ocal)
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        plan.set_colouring(col)
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == want_col.tobytes()
        assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)


@pytest.mark.parametrize("mesh,n,d,perm,env", [("hex27", 2, 7, None, {}), ("hex8", 3, 3, "elements", {"FEA_GATHER_GLOBAL": "1"}),
                                               ("quad4", 5, 2, "nodes", {"FEA_GATHER_GLOBAL": "1"})])
def test_global_gather_fallback(gpu, orc, mesh, n, d, perm, env, monkeypatch):
    """k_gather_global (accumulation in the values array, for plans whose largest row block fits no
    shared-memory gather: here hex27 with d = 7, d * m = 1,323 entries per row block, and forced on
    common shapes): sorted, colour, fused supplier and accumulate bit-exact, repeated nodes too."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    conn, nn = M.make_mesh(mesh, n, perm)
    for collapse in (False, True):
        c2 = M.collapse_elements(conn, np.random.default_rng(5)) if collapse else conn
        ed = M.element_dofs(c2, d)
        P = orc.Pattern.build(c2, nn, d)
        Kh = orc.fill_k(3, c2.shape[0], ed.shape[1])
        want = P.assemble_sequential(ed, Kh)
        col, _ = orc.greedy_colouring(c2, nn)
        K = torch.from_numpy(Kh).cuda()
        with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
            assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
            assert plan.assemble_seeded(3, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
            v = torch.from_numpy(want.copy()).cuda()
            plan.assemble(K, v, strategy="sorted", accumulate=True)
            assert v.cpu().numpy().tobytes() == P.assemble_sequential(ed, Kh, want.copy()).tobytes()
            plan.set_colouring(col)
            assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == P.assemble_coloured(ed, Kh, col).tobytes()
            assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)


@pytest.mark.parametrize("env", [{"FEA_PLAN_NO_FUSED": "1"}])
@pytest.mark.parametrize("mesh,n,d,perm", [("hex8", 4, 3, "elements"), ("tet4", 4, 1, "nodes"), ("hex27", 2, 3, None),
                                           ("quad4", 9, 2, None)])
def test_three_pass_symbolic_route(gpu, orc, mesh, n, d, perm, env, monkeypatch):
    """The separate count / fill / slot-map passes (the route of rows longer than 256 columns and
    of high-valence nodes) give the same pattern and values as the fused pass."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(8, conn.shape[0], ed.shape[1])
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        rp, cs = plan.csr()
        orp, ocs = P.arrays()
        assert np.array_equal(rp, orp) and np.array_equal(cs, ocs)
        got = plan.assemble(torch.from_numpy(Kh).cuda(), strategy="sorted").cpu().numpy()
        assert got.tobytes() == P.assemble_sequential(ed, Kh).tobytes()
        assert close(plan.assemble(torch.from_numpy(Kh).cuda(), strategy="atomic").cpu().numpy(), got)


@pytest.mark.parametrize("mesh,n,d", [("hex8", 3, 3), ("tet4", 2, 2), ("quad4", 4, 2)])
def test_isolated_rows_and_unaligned_k(gpu, orc, mesh, n, d):
    """Rows of nodes no element touches (their CSR rows are empty), and an element-matrix buffer
    that is only 8-byte aligned (the bulk-copy gather needs 16 bytes and hands over to the
    column-node kernel): both bit-exact against the oracle."""
    import torch
    conn, nn = M.make_mesh(mesh, n, "elements")
    extra = 5  # isolated trailing nodes
    ed = M.element_dofs(conn, d)
    P = orc.Pattern.build(conn, nn + extra, d)
    Kh = orc.fill_k(11, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    with gpu.Plan(ed, (nn + extra) * d, dofs_per_node=d) as plan:
        rp, _ = plan.csr()
        assert np.all(np.diff(rp[-extra * d - 1:]) == 0)
        K = torch.from_numpy(Kh).cuda()
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        flat = torch.empty(Kh.size + 1, dtype=torch.float64, device="cuda")
        Ku = flat[1:].view(Kh.shape)
        Ku.copy_(K)
        assert Ku.data_ptr() % 16 == 8
        assert plan.assemble(Ku, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        col, _ = orc.greedy_colouring(conn, nn + extra)
        plan.set_colouring(col)
        want_col = P.assemble_coloured(ed, Kh, col)
        for k in (K, Ku):
            assert plan.assemble(k, strategy="colour").cpu().numpy().tobytes() == want_col.tobytes()


@pytest.mark.parametrize("mesh,n,d,perm", CASES)
def test_atomic_staged_vs_legacy(gpu, orc, mesh, n, d, perm, monkeypatch):
    """The staged atomic kernel (visit-order metadata, cp.async-staged K) and the legacy
    k_scatter<atomic> (FEA_ATOMIC_LEGACY=1, also the path for a K that is not 16-byte
    aligned) both match assemble_sequential within the reference tolerance, and agree
    bitwise with ones K (integer sums are exact in any order)."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(42, E, m)
    want = P.assemble_sequential(ed, Kh)
    ones_want = P.assemble_sequential(ed, np.ones((E, m, m)))
    K = torch.from_numpy(Kh).cuda()
    buf = torch.empty(E * m * m + 1, dtype=torch.float64, device="cuda")
    K_odd = buf[1:].view(E, m, m)  # 8-byte aligned only: legacy kernel
    K_odd.copy_(K)
    for legacy in (False, True):
        if legacy:
            monkeypatch.setenv("FEA_ATOMIC_LEGACY", "1")
        else:
            monkeypatch.delenv("FEA_ATOMIC_LEGACY", raising=False)
        with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
            assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)
            assert close(plan.assemble(K_odd, strategy="atomic").cpu().numpy(), want)
            ones = torch.ones((E, m, m), dtype=torch.float64, device="cuda")
            assert plan.assemble(ones, strategy="atomic").cpu().numpy().tobytes() == ones_want.tobytes()


@pytest.mark.parametrize("seed", range(12))
def test_random_unstructured_meshes(gpu, orc, seed):
    """acceptance.cpp:245-294 (C9, random meshes vs the oracle), on the GPU: random element
    lists over a random node pool — element sizes npe in {3, 4, 6, 8, 10, 20}, d in 1..5,
    random node numbering and element order — so every kernel family and the generic shapes
    (k_gather_node / k_gather_stream / k_scatter) are exercised. Patterns and CRAC arrays
    bit-exact, sorted and colour routes bit-exact, atomics within the reference tolerance."""
    import torch
    rng = np.random.default_rng(1000 + seed)
    npe = int(rng.choice([3, 4, 6, 8, 10, 20]))
    d = int(rng.integers(1, 6))
    nn = int(rng.integers(npe + 2, 200))
    E = int(rng.integers(1, 300))
    # distinct nodes per element, drawn from a local window so rows overlap like a real mesh
    conn = np.empty((E, npe), np.int64)
    for e in range(E):
        lo = int(rng.integers(0, max(1, nn - 3 * npe)))
        conn[e] = lo + rng.choice(min(3 * npe, nn - lo), size=npe, replace=False)
    ed = M.element_dofs(conn, d)
    P = orc.Pattern.build(conn, nn, d)
    rp, cs = P.arrays()
    Kh = orc.fill_k(seed, E, npe * d)
    want = P.assemble_sequential(ed, Kh)
    col, _ = orc.greedy_colouring(conn, nn)
    want_col = P.assemble_coloured(ed, Kh, col)
    K = torch.from_numpy(Kh).cuda()
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        grp, gcs = plan.csr()
        assert np.array_equal(grp, rp) and np.array_equal(gcs, cs)
        for got, exp in zip(plan.crac(), P.crac()):
            assert np.array_equal(got, exp)
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        plan.set_colouring(col)
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == want_col.tobytes()
        assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)


def _check_d1(gpu, orc, conn, nn, ext=None):
    """sorted / colour / accumulate / fused supplier of a d = 1 plan against the oracle"""
    import torch
    ed = M.element_dofs(conn, 1)
    P = orc.Pattern.build(conn, nn, 1)
    Kh = orc.fill_k(5, conn.shape[0], conn.shape[1])
    K = torch.from_numpy(Kh).cuda()
    if ext is None:
        plan, S = gpu.Plan(ed, nn, dofs_per_node=1), P
    else:
        S = orc.Pattern.from_arrays(*ext)
        plan = gpu.Plan.with_pattern(ed, nn, ext[0], ext[1], "csr")
    want = S.assemble_sequential(ed, Kh)
    with plan:
        got = plan.assemble(K, strategy="sorted").cpu().numpy()
        assert got.tobytes() == want.tobytes()
        # accumulate continues the left fold from the existing values
        v = torch.from_numpy(want.copy()).cuda()
        plan.assemble(K, v, strategy="sorted", accumulate=True)
        start = want.copy()
        assert v.cpu().numpy().tobytes() == S.assemble_sequential(ed, Kh, values=start).tobytes()
        col, _ = orc.greedy_colouring(conn, nn)
        plan.set_colouring(col)
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == S.assemble_coloured(ed, Kh, col).tobytes()
        assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)


def test_lane_owned_slots_shapes(gpu, orc):
    """The d = 1, npe = 4 gather with lane-owned slots (k_gather_d1s) and its fall-backs:
    structured tets and quads (every node's link is 3-colourable: compact 4-byte records), a
    fan of 5 tets around an edge (the link of an edge end is an odd wheel: not 3-colourable, the
    plan keeps the shared-memory fold), and a caller's superset pattern (slots no element
    touches stay with lanes 1..3 and keep their start values)."""
    for mesh, n, perm in [("tet4", 5, "nodes"), ("tet4", 3, None), ("quad4", 9, None), ("quad4", 7, "nodes")]:
        conn, nn = M.make_mesh(mesh, n, perm)
        _check_d1(gpu, orc, conn, nn)
    fan = np.array([[0, 1, 2 + i, 2 + (i + 1) % 5] for i in range(5)], np.int64)
    _check_d1(gpu, orc, fan, 7)
    # fan glued to a structured block: one plan mixes colourable and non-colourable nodes
    conn, nn = M.make_mesh("tet4", 2, None)
    _check_d1(gpu, orc, np.concatenate([conn, fan + nn]), nn + 7)
    # superset pattern on a small tet mesh: one extra column per row (rows stay <= 16 nodes)
    conn, nn = M.make_mesh("tet4", 2, "nodes")
    P = orc.Pattern.build(conn, nn, 1)
    rp, cs = P.arrays()
    rng = np.random.default_rng(9)
    rows = []
    for r in range(nn):
        have = cs[rp[r]:rp[r + 1]]
        extra = rng.choice(np.setdiff1d(np.arange(nn), have), size=1)
        rows.append(np.unique(np.concatenate([have, extra])))
    srp = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    _check_d1(gpu, orc, conn, nn, ext=(srp, np.concatenate(rows).astype(np.int64)))


@pytest.mark.parametrize("env", [{"FEA_PATCH_TICKETS": "1"}, {"FEA_PATCH_TICKETS": "1", "FEA_PATCH_TILE": "2"},
                                 {"FEA_PATCH_STATIC": "1", "FEA_PATCH_TILE": "3"}, {"FEA_PATCH_NO_TILES": "1"},
                                 {"FEA_PATCH_HOST_SWEEP": "1"}, {"FEA_PATCH_HOST_SWEEP": "1", "FEA_PATCH_TILE": "2"}])
@pytest.mark.parametrize("n,perm", [(8, None), (7, None), (6, "elements")])
def test_atomic_patch_schedules(gpu, orc, env, n, perm, monkeypatch):
    """k_atomic_patch under every patch schedule: tickets / grid stride, lattice tiles of several
    sizes (forced on a small lexicographic mesh, where the detection finds s1 = n/2, s2 = (n/2)^2)
    or the sequence order; patches found on the device as node stars (even n) or by the host sweep
    (odd n, or forced). Any order is a valid atomic assembly: within the reference tolerance of
    the sequential result, and bitwise with ones (every sum is exact)."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    conn, nn, ed, n_rows = problem("hex8", n, 3, perm)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, 3)
    Kh = orc.fill_k(3, E, m)
    want = P.assemble_sequential(ed, Kh)
    ones = np.ones_like(Kh)
    want1 = P.assemble_sequential(ed, ones)
    with gpu.Plan(ed, n_rows, dofs_per_node=3) as plan:
        for _ in range(2):  # the second launch takes the next ticket counter of the ring
            assert close(plan.assemble(torch.from_numpy(Kh).cuda(), strategy="atomic").cpu().numpy(), want)
        got1 = plan.assemble(torch.from_numpy(ones).cuda(), strategy="atomic").cpu().numpy()
        assert got1.tobytes() == want1.tobytes()


@pytest.mark.parametrize("dims,perm_nodes", [((2, 2, 40), False), ((4, 2, 6), True), ((6, 4, 2), False), ((3, 4, 4), False)])
def test_atomic_star_patches_boxes(gpu, orc, dims, perm_nodes, monkeypatch, capfd):
    """Patches found on the device as node stars on non-cubic boxes: a thin bar (a long chain of
    selection rounds), permuted node ids (another independent set, still a tiling or else the host
    sweep), an odd direction (stars leave elements over: host sweep). Atomic within the reference
    tolerance, bitwise with ones."""
    import torch
    monkeypatch.setenv("FEA_PATCH_DEBUG", "1")
    conn, nn = M.hex8_box(*dims)
    if perm_nodes:
        conn = np.random.default_rng(3).permutation(nn)[conn]
    ed = M.element_dofs(conn, 3)
    P = orc.Pattern.build(conn, nn, 3)
    Kh = orc.fill_k(6, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    ones = np.ones_like(Kh)
    with gpu.Plan(ed, nn * 3, dofs_per_node=3) as plan:
        assert close(plan.assemble(torch.from_numpy(Kh).cuda(), strategy="atomic").cpu().numpy(), want)
        got1 = plan.assemble(torch.from_numpy(ones).cuda(), strategy="atomic").cpu().numpy()
        assert got1.tobytes() == P.assemble_sequential(ed, ones).tobytes()
    err = capfd.readouterr().err
    if not perm_nodes and all(x % 2 == 0 for x in dims):
        assert "(stars)" in err, err  # lexicographic even boxes are tiled by the stars
    if any(x % 2 for x in dims):
        assert "(stars)" not in err, err


@pytest.mark.parametrize("env", [{}, {"FEA_PATCH_TICKETS": "1"}, {"FEA_STRIP_LONG": "0"}, {"FEA_ATOMIC_NO_STRIP": "1"}])
@pytest.mark.parametrize("mesh,n,perm", [("tet4", 5, "nodes"), ("tet4", 4, "elements"), ("quad4", 13, "elements"),
                                         ("quad4", 9, None)])
def test_atomic_strip_paths(gpu, orc, env, mesh, n, perm, monkeypatch):
    """k_atomic_strip (npe = 4, d = 1): consecutive K rows (one bulk copy per strip) and permuted
    elements (a copy per element), strips by grid stride or by ticket, both pair orders, a
    partial last strip, a row-partitioned plan, accumulate; against the sequential result within
    the reference tolerance, bitwise with ones."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    conn, nn, ed, n_rows = problem(mesh, n, 1, perm)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, 1)
    Kh = orc.fill_k(4, E, m)
    want = P.assemble_sequential(ed, Kh)
    ones = np.ones_like(Kh)
    want1 = P.assemble_sequential(ed, ones)
    K = torch.from_numpy(Kh).cuda()
    with gpu.Plan(ed, n_rows, dofs_per_node=1) as plan:
        for _ in range(2):
            assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)
        assert plan.assemble(torch.from_numpy(ones).cuda(), strategy="atomic").cpu().numpy().tobytes() == want1.tobytes()
        v = torch.from_numpy(want1.copy()).cuda()  # accumulate onto existing values (exact with ones)
        plan.assemble(torch.from_numpy(ones).cuda(), v, strategy="atomic", accumulate=True)
        assert v.cpu().numpy().tobytes() == (2 * want1).tobytes()
    rp, _ = P.arrays()
    lo, hi = n_rows // 3, (2 * n_rows) // 3
    with gpu.Plan(ed, n_rows, dofs_per_node=1, row_range=(lo, hi)) as plan:
        got = plan.assemble(K, strategy="atomic").cpu().numpy()
        assert close(got, want[rp[lo]:rp[hi]])


KERNEL_SWITCHES = ["FEA_SLOT_NO_FIXED", "FEA_CN_NO_RECORDS", "FEA_D1_NO_DIRECT", "FEA_D1_NO_VEC",
                   "FEA_GATHER_NO_SLOT", "FEA_GATHER_NO_CN", "FEA_D1_NO_LANE", "FEA_D1_REC8",
                   "FEA_D1_NO_LANE,FEA_D1_NO_DIRECT", "FEA_GATHER_GLOBAL"]


@pytest.mark.parametrize("switch", KERNEL_SWITCHES)
@pytest.mark.parametrize("mesh,n,d,perm", [("hex8", 3, 3, "elements"), ("tet4", 4, 1, "nodes"),
                                            ("hex27", 2, 3, None)])
def test_kernel_switches_same_bits(gpu, orc, switch, mesh, n, d, perm, monkeypatch):
    """Every A/B switch selects another kernel of the same route: the sorted and
    colour routes and the fused supplier stay bit-identical to the oracle / the default path."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(42, E, m)
    want = P.assemble_sequential(ed, Kh)
    col, _ = orc.greedy_colouring(conn, nn)
    want_col = P.assemble_coloured(ed, Kh, col)
    K = torch.from_numpy(Kh).cuda()
    for sw in switch.split(","):  # read when the plan is created
        monkeypatch.setenv(sw, "1")
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes()
        plan.set_colouring(col)
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == want_col.tobytes()
        Ks = gpu.fill_seeded_k(E, m, 11)
        ref = plan.assemble(Ks, strategy="sorted").cpu().numpy()
        assert plan.assemble_seeded(11, strategy="sorted").cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("mesh,n,d,perm", [("hex8", 3, 3, "elements"), ("tet4", 4, 1, "nodes"),
                                            ("hex27", 2, 3, None)])
def test_cuda_graph_replay(gpu, orc, mesh, n, d, perm):
    """After one warm-up call per route (which builds the lazily created plan tables), the
    assembly is stream-ordered with no host synchronisation: it can be captured in a CUDA graph
    and replayed (the launch-bound inner loop of a Newton / time-stepping caller)."""
    import torch
    conn, nn, ed, n_rows = problem(mesh, n, d, perm)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(42, E, m)
    want = P.assemble_sequential(ed, Kh)
    K = torch.from_numpy(Kh).cuda()
    with gpu.Plan(ed, n_rows, dofs_per_node=d) as plan:
        plan.set_colouring(plan.greedy_colouring()[0])
        for strategy in ("sorted", "colour", "atomic"):
            v = torch.zeros(plan.nnz, dtype=torch.float64, device="cuda")
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                plan.assemble(K, v, strategy=strategy, stream=s)  # warm-up: lazy tables
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                v.zero_()
                plan.assemble(K, v, strategy=strategy, accumulate=True, stream=s)
            v.fill_(7.0)
            g.replay()
            torch.cuda.synchronize()
            got = v.cpu().numpy()
            if strategy == "atomic":
                assert close(got, want)
            elif strategy == "sorted":
                assert got.tobytes() == want.tobytes()


def test_binding_rejects_bad_buffers(gpu):
    """Plan.assemble* check dtype, size and device of K / values before raw pointers cross the
    ABI (a float32 or short K would be read out of bounds by the kernels)."""
    import torch
    conn, nn, ed, n_rows = problem("hex8", 2, 3, None)
    E, m = ed.shape
    with gpu.Plan(ed, n_rows, dofs_per_node=3) as plan:
        good = gpu.fill_seeded_k(E, m, 1)
        v = plan.assemble(good)
        for K in (good.float(), good[:-1], good.cpu()):
            with pytest.raises(AssertionError):
                plan.assemble(K)
        with pytest.raises(AssertionError):
            plan.assemble(good, v[:-1])
        with pytest.raises(AssertionError):
            plan.assemble_host(good.cpu().numpy().astype(np.float32))
        with pytest.raises(AssertionError):
            plan.assemble_seeded(1, v[:-1])


def test_pinned_host_buffers_end_to_end(gpu, orc):
    """hostmem.pinned_empty (cudaHostRegister'ed numpy arrays) through the pipelined host path:
    bit-exact vs the oracle; the registration is dropped with the array."""
    import gc
    from paper_2012_00585_b200.hostmem import pinned_empty
    conn, nn, ed, n_rows = problem("hex8", 5, 3, None)
    P = orc.Pattern.build(conn, nn, 3)
    E, m = ed.shape
    Kh = pinned_empty((E, m, m))
    Kh[...] = orc.fill_k(11, E, m)
    vh = pinned_empty((P.nnz,))
    with gpu.Plan(ed, n_rows, dofs_per_node=3) as plan:
        plan.set_host_windows(4)
        plan.assemble_host(Kh, vh, strategy="sorted")
        assert vh.tobytes() == P.assemble_sequential(ed, Kh).tobytes()
    del Kh, vh
    gc.collect()
