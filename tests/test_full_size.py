"""GPU parity at the BASELINE sizes (configs 1-5), through the C ABI, against the CPU oracle.

The reference pins exact integer results and cross-method equality at scale (exact NNZ,
acceptance.cpp:109-136; bitwise cross-method equality, :180-199; dense-oracle equivalence,
:245-294). Here every BASELINE configuration is checked at its full size:

  configs 1-3  whole pattern + CRAC arrays bit-exact vs the oracle's build_pattern /
               build_crac_arrays (pattern.cpp:24-108, formats.cpp:21-41); the device greedy
               colouring equal to greedy_colouring (colouring.cpp:24-75); sorted, fused-supplier,
               colour and colour-pass values bit-exact vs assemble_sequential /
               assemble_coloured_vectorized; atomic within 1e-12; ones-K exact conservation
  config 4     whole pattern + CRAC bit-exact; values on sampled node rows (restricted oracle)
  config 5     NNZ 4,092,809,481 > 2^31: the WHOLE int64 CSR and CRAC row pointers against the
               restricted oracle's row counts / runs, the greedy colouring, and columns, CRAC
               pairs and values (sorted, colour, fused bit-exact; atomic within 1e-12) of 4,096+
               sampled node rows spread over the whole int64 offset range
"""
import numpy as np
import pytest

from paper_2012_00585_b200 import meshgen as M

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 1e-12  # test_assembly.cpp:236


def close(a, b, tol=TOL):
    return bool(np.all(np.abs(a - b) <= tol * np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))


def close_t(a, b, tol=TOL):
    import torch
    return bool(torch.all((a - b).abs() <= tol * torch.maximum(torch.maximum(a.abs(), b.abs()),
                                                               torch.ones_like(a))).item())


@pytest.mark.timeout(600)
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_config_full_oracle(gpu, orc, cfg):
    import torch
    conn, nn, d = M.config_mesh(cfg)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, d)
    if M.CONFIGS[cfg]["perm"] != "nodes":
        assert P.nnz == M.closed_form_nnz(M.CONFIGS[cfg]["mesh"], M.CONFIGS[cfg]["n"], d)
    ocol, onc = orc.greedy_colouring(conn, nn)
    Kh = orc.fill_k(42, E, m)
    want = P.assemble_sequential(ed, Kh)
    want_c = P.assemble_coloured(ed, Kh, ocol)
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        assert (plan.n_rows, plan.nnz, plan.n_runs) == (P.n_rows, P.nnz, P.n_runs)
        rp, cs = plan.csr()
        orp, ocs = P.arrays()
        assert np.array_equal(rp, orp) and np.array_equal(cs, ocs)
        cp, ca = plan.crac()
        ocp, oca = P.crac()
        assert np.array_equal(cp, ocp) and np.array_equal(ca, oca)
        del rp, cs, cp, ca, orp, ocs, ocp, oca
        col, nc = plan.greedy_colouring()
        assert nc == onc and np.array_equal(col, ocol)
        plan.set_colouring(col)
        K = gpu.fill_seeded_k(E, m, 42)
        assert torch.equal(K, torch.from_numpy(Kh).cuda())
        del Kh
        wb = want.tobytes()
        assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == wb
        assert plan.assemble_seeded(42, strategy="sorted").cpu().numpy().tobytes() == wb
        assert plan.assemble(K, strategy="colour").cpu().numpy().tobytes() == want_c.tobytes()
        assert plan.assemble(K, strategy="colour_passes").cpu().numpy().tobytes() == want_c.tobytes()
        assert close(plan.assemble(K, strategy="atomic").cpu().numpy(), want)
        K.fill_(1.0)  # ones: exact conservation, every route bitwise equal (acceptance.cpp:180-199)
        ones = plan.assemble(K, strategy="sorted")
        assert float(ones.sum().item()) == float(E * m * m)
        for s in ("atomic", "colour", "colour_passes"):
            assert torch.equal(plan.assemble(K, strategy=s), ones)


def sampled_nodes(nn, n_sample=4096, seed=5):
    rng = np.random.default_rng(seed)
    pick = np.concatenate([[0, 1, nn // 2, nn - 2, nn - 1], rng.integers(0, nn, size=n_sample)])
    return np.unique(pick)


def row_index(rp, nodes, cnt, d):
    """Value positions of the selected nodes' rows: [node][k][slot] -> flat index array."""
    idx = []
    for i, v in enumerate(nodes):
        for k in range(d):
            r = v * d + k
            idx.append(np.arange(rp[r], rp[r + 1], dtype=np.int64))
            assert rp[r + 1] - rp[r] == d * cnt[i]
    return np.concatenate(idx)


def expected_rows(vals, cnt, d):
    return np.concatenate([vals[i, k, :d * cnt[i]] for i in range(len(cnt)) for k in range(d)])


def check_sampled(gpu, plan, K_fn, conn, nn, d, seed, rp, A, ocol, full_colour_check=True):
    """Columns, CRAC pairs and values of sampled node rows against the restricted oracle."""
    import torch
    nodes = sampled_nodes(nn)
    cnt, cols, vals = A.node_rows(nodes, d, seed)
    _, _, vals_c = A.node_rows(nodes, d, seed, colour_of=ocol)
    idx = row_index(rp, nodes, cnt, d)
    idx_d = torch.from_numpy(idx).cuda()
    # columns of the sampled rows (device CSR expansion, int64)
    rp_d, cs_d = plan.csr_device()
    got_cols = cs_d[idx_d].cpu().numpy()
    want_cols = np.concatenate([np.repeat(cols[i, :cnt[i]] * d, d) + np.tile(np.arange(d), cnt[i])
                                for i in range(len(nodes)) for _ in range(d)])
    assert np.array_equal(got_cols, want_cols)
    del rp_d, cs_d
    # CRAC pairs of the sampled rows: (column start, values position) per run (formats.cpp:21-41)
    cp_d, ca_d = plan.crac_device()
    cp = cp_d.cpu().numpy()
    for i, v in enumerate(nodes[:512]):
        for k in range(d):
            r = v * d + k
            pairs = ca_d[cp[r]:cp[r + 1]].cpu().numpy().reshape(-1, 2)
            c = cols[i, :cnt[i]]
            starts = np.flatnonzero(np.concatenate([[True], np.diff(c) != 1]))
            assert np.array_equal(pairs[:, 0], c[starts] * d)
            assert np.array_equal(pairs[:, 1], rp[r] + starts * d)
    assert int(ca_d[-1].item()) == plan.nnz and int(ca_d[-2].item()) == 0
    del cp_d, ca_d
    torch.cuda.empty_cache()
    want = expected_rows(vals, cnt, d)
    want_c = expected_rows(vals_c, cnt, d)
    K = K_fn()
    values = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.assemble(K, values, strategy="sorted")
    assert values[idx_d].cpu().numpy().tobytes() == want.tobytes()
    if full_colour_check:
        plan.assemble(K, values, strategy="colour")
        assert values[idx_d].cpu().numpy().tobytes() == want_c.tobytes()
    values.zero_()
    plan.assemble(K, values, strategy="atomic", accumulate=True)
    assert close(values[idx_d].cpu().numpy(), want)
    del K
    torch.cuda.empty_cache()
    plan.assemble_seeded(seed, values, strategy="sorted")
    assert values[idx_d].cpu().numpy().tobytes() == want.tobytes()
    return values


@pytest.mark.timeout(900)
def test_config4_full_pattern_sampled_values(gpu, orc):
    conn, nn, d = M.config_mesh(4)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    P = orc.Pattern.build(conn, nn, d)
    assert P.nnz == M.closed_form_nnz("hex27", 48, d) == 513_599_625
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        rp, cs = plan.csr()
        orp, ocs = P.arrays()
        assert np.array_equal(rp, orp) and np.array_equal(cs, ocs)
        del cs, ocs
        cp, ca = plan.crac()
        ocp, oca = P.crac()
        assert np.array_equal(cp, ocp) and np.array_equal(ca, oca)
        del cp, ca, ocp, oca, P
        ocol, onc = orc.greedy_colouring(conn, nn)
        col, nc = plan.greedy_colouring()
        assert nc == onc and np.array_equal(col, ocol)
        plan.set_colouring(col)
        A = orc.Adjacency(conn, nn)
        check_sampled(gpu, plan, lambda: gpu.fill_seeded_k(E, m, 42), conn, nn, d, 42, rp, A, ocol)


@pytest.mark.timeout(900)
def test_config5_int64_offsets_row_pointers_and_sampled_rows(gpu, orc):
    """BASELINE config 5 on one GPU: NNZ 4,092,809,481 needs int64 value offsets. The whole
    CSR/CRAC row pointers come from the restricted oracle's per-node counts (an independent
    scan), so a wrong int64 row start cannot hide behind a cross-route comparison."""
    import torch
    n, d = 256, 3
    conn, nn = M.hex8_structured(n)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    A = orc.Adjacency(conn, nn)
    orp, ocp = A.row_ptrs(d)
    assert orp[-1] == M.closed_form_nnz("hex8", n, d) == 4_092_809_481 > 2 ** 31
    ocol, onc = orc.greedy_colouring(conn, nn)
    with gpu.Plan(ed, nn * d, dofs_per_node=d) as plan:
        del ed
        assert plan.nnz == orp[-1] and plan.n_runs == d * (n + 1) * (3 * n + 1) ** 2 == ocp[-1] // 2
        rp = plan.row_ptr()
        assert np.array_equal(rp, orp)
        cp_d, _ = plan.crac_device()
        assert np.array_equal(cp_d.cpu().numpy(), ocp)
        del cp_d
        col, nc = plan.greedy_colouring()
        assert nc == onc == 8 and np.array_equal(col, ocol)
        plan.set_colouring(col)
        del col
        values = check_sampled(gpu, plan, lambda: gpu.fill_seeded_k(E, m, 42), conn, nn, d, 42, rp, A, ocol)
        # the last value slot lives beyond 2^32 bytes * 8: written, finite
        assert np.isfinite(values[-1].item()) and values[-1].item() != 0.0
        del values
        torch.cuda.empty_cache()
