"""CPU: pin the oracle (oracle/oracle.c) to the reference's golden vectors and to the
compiled reference library. No GPU needed.

Golden sources: the reference's own tests (test_formats.cpp, test_mesh.cpp, test_pattern.cpp,
test_assembly.cpp, acceptance.cpp — values restated here with file:line) and fixtures made by
tests/golden/make_golden.py from the unmodified reference library.
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from paper_2012_00585_b200 import meshgen as M

GOLD = Path(__file__).resolve().parent / "golden"
CASES = {
    "quad4_n6_d1": ("quad4", 6, 1, None),
    "quad4_n5_d2_nodeperm": ("quad4", 5, 2, "nodes"),
    "hex8_n3_d3_elemperm": ("hex8", 3, 3, "elements"),
    "tet4_n3_d1_nodeperm": ("tet4", 3, 1, "nodes"),
    "hex27_n2_d3": ("hex27", 2, 3, None),
    "hex8_n4_d1": ("hex8", 4, 1, None),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gold_case(name):
    g = np.load(GOLD / f"{name}.npz")
    if name.startswith("refdofmap"):
        conn = np.load(GOLD / f"{name}_conn.npy")
    else:
        mesh, n, d, perm = CASES[name]
        conn, _ = M.make_mesh(mesh, n, perm)
    assert sha(conn) == str(g["conn_sha"]), "mesh generator changed"
    return g, conn, int(g["n_nodes"]), int(g["d"])


# ---- Fig. 1 6x6 example (test_formats.cpp:31-109, acceptance.cpp:57-96) ----

FIG1_ROWS = [[0, 1], [0, 1], [1, 2, 4, 5], [2, 3, 4], [3, 4, 5], [1, 2, 3, 4]]


def test_fig1_csr_crac_arrays(orc):
    rp = np.concatenate([[0], np.cumsum([len(r) for r in FIG1_ROWS])])
    cs = np.concatenate(FIG1_ROWS)
    P = orc.Pattern.from_arrays(rp, cs)
    assert list(rp + 1) == [1, 3, 5, 9, 12, 15, 19]                     # test_formats.cpp:54
    assert P.n_runs == 7                                                  # :63
    crp, ca = P.crac()
    assert list(crp) == [0, 2, 4, 8, 10, 12, 14]                          # :65
    assert list(ca[:-2]) == [0, 0, 0, 2, 1, 4, 4, 6, 2, 8, 3, 11, 1, 14]  # :69-70
    assert ca[-1] == 18 and ca[-2] == 0                                   # :71
    g = np.load(GOLD / "fig1.npz")
    assert np.array_equal(crp, g["crac_ptr"]) and np.array_equal(ca, g["col_align"])
    # lookups: (3,6) at 8 (1-based), (6,2) at 15, (1,6) absent, below first run absent
    assert P.locate(2, 5) == 7 and orc.locate_crac(crp, ca, 2, 5) == 7    # :78-85
    assert P.locate(5, 1) == 14 and orc.locate_crac(crp, ca, 5, 1) == 14  # :96-101
    assert P.locate(0, 5) == -1 and orc.locate_crac(crp, ca, 0, 5) == -1  # :90-93
    assert orc.locate_crac(crp, ca, 2, 0) == -1 and orc.locate_crac(crp, ca, 4, 0) == -1  # :104-107
    for r, c, want_csr, want_crac in g["lookups"]:
        assert P.locate(r, c) == want_csr
        assert orc.locate_crac(crp, ca, r, c) == want_crac


def test_empty_pattern_and_empty_rows(orc):
    """test_formats.cpp:111-139."""
    P = orc.Pattern.from_arrays(np.array([0]), np.array([], np.int64))
    crp, ca = P.crac()
    assert list(crp) == [0] and list(ca) == [0, 0]
    rows = [[1, 2], [], [0, 3], [], [], [2]]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    P = orc.Pattern.from_arrays(rp, np.concatenate([np.array(r, np.int64) for r in rows]))
    crp, ca = P.crac()
    for c in range(6):
        assert P.locate(1, c) == -1 and orc.locate_crac(crp, ca, 1, c) == -1
        assert orc.locate_crac(crp, ca, 4, c) == -1
    assert orc.locate_crac(crp, ca, 2, 0) == P.locate(2, 0)
    assert orc.locate_crac(crp, ca, 5, 2) == 4


def test_linear_and_binary_search_agree(orc):
    """test_formats.cpp:176-188: rows above kLinearSearchMax (30) use binary search."""
    rng = np.random.default_rng(5)
    rows = [np.sort(rng.choice(200, size=s, replace=False)) for s in (5, 29, 30, 31, 60, 120)]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    P = orc.Pattern.from_arrays(rp, np.concatenate(rows))
    for r, row in enumerate(rows):
        for c in range(200):
            hit = np.searchsorted(row, c)
            want = rp[r] + hit if hit < len(row) and row[hit] == c else -1
            assert P.locate(r, c) == want


# ---- RLE (test_mesh.cpp:210-271, acceptance.cpp:98-107) ----

def test_rle_fixture(orc):
    flat = [52, 53, 54, 55, 96, 97, 98, 99, 100, 101, 102, 103, 48, 49, 50, 51]
    assert orc.encode_runs(flat) == [(52, 4), (96, 8), (48, 4)]
    assert orc.encode_runs([7]) == [(7, 1)]
    rng = np.random.default_rng(42)
    for _ in range(20):
        flat = rng.integers(0, 20, size=12)
        runs = orc.encode_runs(flat)
        assert [s + k for s, ln in runs for k in range(ln)] == list(flat)
        assert all(a[0] + a[1] != b[0] for a, b in zip(runs, runs[1:]))


# ---- exact NNZ tables (test_pattern.cpp:63-97, acceptance.cpp:109-165) ----

def test_pattern_fixture_nnz(orc):
    conn, nn = M.quad4_structured(6)
    assert orc.Pattern.build(conn, nn, 1).nnz == 361
    conn, nn = M.quad4_structured(1)
    P = orc.Pattern.build(conn, nn, 1)
    assert P.n_rows == 4 and P.nnz == 16


def test_h_suite_nnz_768(orc):
    """acceptance.cpp:111: structured 768x768, p=1, d=1 -> 5313025; DOF axis :126."""
    conn, nn = M.quad4_structured(768)
    assert orc.Pattern.build(conn, nn, 1).nnz == 5313025
    assert [M.quad4_structured(n)[1] for n in (6, 12, 24, 48, 96, 192, 384, 768)] == \
        [49, 169, 625, 2401, 9409, 37249, 148225, 591361]


def test_d_scaling_identities(orc):
    """acceptance.cpp:138-165: nnz(d) = d^2 nnz(1); n_ca(d) = d (n_ca(1) - 2) + 2."""
    for n in (2, 6, 48):
        conn, nn = M.quad4_structured(n)
        base = orc.Pattern.build(conn, nn, 1)
        ca1 = 2 * base.n_runs + 2
        for d in (2, 4, 8):
            P = orc.Pattern.build(conn, nn, d)
            assert P.nnz == d * d * base.nnz
            assert 2 * P.n_runs + 2 == d * (ca1 - 2) + 2
    assert orc.Pattern.build(*M.quad4_structured(192), 4).nnz == 5326864   # acceptance.cpp:113
    assert orc.Pattern.build(*M.quad4_structured(192), 8).nnz == 21307456  # :117


def test_ref_dofmap_p_suite_nnz(orc, ref_lib):
    """acceptance.cpp:112-116 with the reference's own p-refined DOF numbering."""
    conn, nn = ref_lib.ref_structured_element_nodes(48, 8, 1)
    assert orc.Pattern.build(conn, nn, 1).nnz == 14753281
    conn, nn = ref_lib.ref_structured_element_nodes(48, 4, 1)
    assert orc.Pattern.build(conn, nn, 4).nnz == 21270544
    assert ref_lib.ref_speed_factor(117074.0, 20489.3) == pytest.approx(5.713, abs=1e-3)  # C7


def test_storage_factor_p_refinement(orc, ref_lib):
    """acceptance.cpp:296-332: gamma(p=8) < 0.25 < gamma(p=1), gamma = (2 runs + 2) / nnz."""
    g = {}
    for p in (1, 3, 8):
        conn, nn = ref_lib.ref_structured_element_nodes(48, p, 1)
        P = orc.Pattern.build(conn, nn, 1)
        g[p] = (2 * P.n_runs + 2) / P.nnz
    assert g[8] < 0.25 < g[1] and g[8] < g[3] < g[1]


def test_closed_form_3d(orc):
    """SURVEY.md §8.0 closed forms for our 3D meshes."""
    for mesh, ns in (("hex8", (1, 2, 3, 5)), ("hex27", (1, 2, 3)), ("tet4", (1, 2, 4))):
        for n in ns:
            for d in (1, 3):
                conn, nn = M.make_mesh(mesh, n)
                assert orc.Pattern.build(conn, nn, d).nnz == M.closed_form_nnz(mesh, n, d)
    conn, nn = M.hex8_structured(5)
    assert orc.Pattern.build(conn, nn, 3).n_runs == 3 * 6 * 16 * 16  # d(n+1)(3n+1)^2


# ---- colouring (acceptance.cpp:167-178, test_colouring.cpp) ----

def test_structured_colouring_four_colours(orc):
    for n in (2, 6, 48, 192):
        conn, nn = M.quad4_structured(n)
        col, nc = orc.greedy_colouring(conn, nn)
        assert nc == 4
        assert all(np.count_nonzero(col == c) * 4 == n * n for c in range(4))


def test_colouring_valid(orc):
    for mesh, n, perm in (("hex8", 4, "elements"), ("tet4", 3, "nodes"), ("hex27", 2, None)):
        conn, nn = M.make_mesh(mesh, n, perm)
        col, nc = orc.greedy_colouring(conn, nn)
        for c in range(nc):
            nodes = conn[col == c].reshape(-1)
            assert len(np.unique(nodes)) == len(nodes)


# ---- golden fixtures from the reference library ----

@pytest.mark.parametrize("name", list(CASES) + ["refdofmap_n4_p3_d2"])
def test_oracle_matches_reference_fixtures(orc, name):
    g, conn, nn, d = gold_case(name)
    P = orc.Pattern.build(conn, nn, d)
    rp, cs = P.arrays()
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(cs, g["cols"])
    crp, ca = P.crac()
    assert np.array_equal(crp, g["crac_ptr"]) and np.array_equal(ca, g["col_align"])
    col, nc = orc.greedy_colouring(conn, nn)
    assert np.array_equal(col, g["colour_of"]) and nc == int(g["n_colours"])
    ed = M.element_dofs(conn, d)
    K = orc.fill_k(42, conn.shape[0], ed.shape[1])
    assert sha(K) == str(g["k_sha"]), "K generator changed"
    assert P.assemble_sequential(ed, K).tobytes() == g["values_seq"].tobytes()
    assert P.assemble_coloured(ed, K, col).tobytes() == g["values_colour"].tobytes()
    ones = P.assemble_sequential(ed, np.ones_like(K))
    assert ones.tobytes() == g["values_ones"].tobytes()
    assert ones.sum() == conn.shape[0] * ed.shape[1] ** 2   # verify.cpp:85-100


def test_oracle_matches_live_reference_random(orc, ref_lib):
    """Differential test against the compiled reference on random permuted meshes."""
    rng = np.random.default_rng(2026)
    for trial in range(12):
        mesh = ["quad4", "hex8", "tet4", "hex27"][trial % 4]
        n = int(rng.integers(1, 4 if mesh != "quad4" else 7))
        d = int(rng.integers(1, 4))
        perm = [None, "nodes", "elements"][trial % 3]
        conn, nn = M.make_mesh(mesh, n, perm, seed=int(rng.integers(1 << 30)))
        R = ref_lib.RefProblem(conn, nn, d)
        P = orc.Pattern.build(conn, nn, d)
        rp, cs = P.arrays()
        rrp, rcs = R.pattern()
        assert np.array_equal(rp, rrp) and np.array_equal(cs, rcs)
        ed = M.element_dofs(conn, d)
        K = orc.fill_k(int(rng.integers(1 << 30)), conn.shape[0], ed.shape[1])
        assert P.assemble_sequential(ed, K).tobytes() == R.assemble(K, "seq", "crac").tobytes()
        col, _ = R.greedy_colouring(conn.shape[0])
        assert P.assemble_coloured(ed, K, col).tobytes() == \
            R.assemble(K, "colour-vec", "csr", threads=3, colour_of=col).tobytes()
        atomic = R.assemble(K, "atomic", "csr", threads=4)
        want = P.assemble_sequential(ed, K)
        assert np.all(np.abs(atomic - want) <= 1e-12 * np.maximum(np.maximum(abs(atomic), abs(want)), 1))


def test_dense_oracle_equivalence(orc):
    """acceptance.cpp:245-294 (criterion 9): sequential assembly == dense accumulation."""
    rng = np.random.default_rng(20260809)
    for trial in range(30):
        mesh = ["quad4", "hex8", "tet4"][trial % 3]
        conn, nn = M.make_mesh(mesh, int(rng.integers(1, 4)), ["nodes", None][trial % 2],
                               seed=int(rng.integers(1000)))
        d = int(rng.integers(1, 3))
        ed = M.element_dofs(conn, d)
        n_rows = nn * d
        integer_k = trial % 3 == 0
        K = np.ones((conn.shape[0], ed.shape[1], ed.shape[1])) if integer_k else \
            orc.fill_k(trial, conn.shape[0], ed.shape[1])
        dense = np.zeros((n_rows, n_rows))
        for e in range(conn.shape[0]):
            dense[np.ix_(ed[e], ed[e])] += K[e]
        P = orc.Pattern.build(conn, nn, d)
        v = P.assemble_sequential(ed, K)
        rp, cs = P.arrays()
        got = np.zeros((n_rows, n_rows))
        for r in range(n_rows):
            got[r, cs[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
        if integer_k:
            assert np.array_equal(got, dense)
        else:
            assert np.all(np.abs(got - dense) <= 1e-12 * np.maximum(np.abs(dense), 1.0))


def test_missing_entry_reports_first_coefficient(orc):
    """test_assembly.cpp:122-141: pattern of the first element only, four assembled."""
    conn, nn = M.quad4_structured(2)
    P = orc.Pattern.build(conn[:1], nn, 1)
    with pytest.raises(orc.MissingEntry) as ei:
        P.assemble_sequential(M.element_dofs(conn, 1), np.ones((4, 4, 4)))
    e, r, c = ei.value.args[0]
    assert e == 1 and r == conn[1, 0]


def test_seeded_k_exact_and_symmetric(orc):
    K = orc.fill_k(42, 5, 24)
    assert np.array_equal(K, np.swapaxes(K, 1, 2))
    assert K.min() >= -1.0 and K.max() < 1.0
    # (h>>11) * 2^-53 * 2 - 1 is exact: every value is a multiple of 2^-52
    assert np.all(np.ldexp(K + 1.0, 52) == np.round(np.ldexp(K + 1.0, 52)))


def test_degenerate_elements_match_live_reference(orc, ref_lib):
    rng = np.random.default_rng(77)
    for trial, (mesh, n, d) in enumerate([("quad4", 4, 1), ("quad4", 3, 2), ("hex8", 2, 3),
                                           ("tet4", 2, 1), ("hex8", 2, 1)]):
        conn, nn = M.make_mesh(mesh, n, "nodes" if trial % 2 else None, seed=trial)
        conn = M.collapse_elements(conn, rng)
        R = ref_lib.RefProblem(conn, nn, d)
        P = orc.Pattern.build(conn, nn, d)
        rp, cs = P.arrays()
        rrp, rcs = R.pattern()
        assert np.array_equal(rp, rrp) and np.array_equal(cs, rcs)
        ed = M.element_dofs(conn, d)
        K = orc.fill_k(trial, conn.shape[0], ed.shape[1])
        assert P.assemble_sequential(ed, K).tobytes() == R.assemble(K, "seq", "csr").tobytes()
        col, _ = R.greedy_colouring(conn.shape[0])
        assert P.assemble_coloured(ed, K, col).tobytes() == \
            R.assemble(K, "colour-vec", "csr", threads=2, colour_of=col).tobytes()
        ones = P.assemble_sequential(ed, np.ones_like(K))
        assert ones.sum() == conn.shape[0] * ed.shape[1] ** 2


# ---- restricted oracle (config 5 scale: whole row pointers + selected rows) ----

@pytest.mark.parametrize("name", list(CASES) + ["refdofmap_n4_p3_d2"])
def test_restricted_oracle_matches_reference_fixtures(orc, name):
    """orc.Adjacency (the full-size check of config 5, NNZ 4.09e9) against arrays made by the
    unmodified reference: whole CSR / CRAC row pointers, and every node's rows (columns,
    sequential and colour-vec values with the seeded supplier) bit for bit."""
    g, conn, nn, d = gold_case(name)
    A = orc.Adjacency(conn, nn)
    rp, cp = A.row_ptrs(d, threads=3)
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(cp, g["crac_ptr"])
    nodes = np.arange(nn)
    for colour, want in ((None, g["values_seq"]), (g["colour_of"], g["values_colour"])):
        cnt, cols, vals = A.node_rows(nodes, d, 42, colour_of=colour)
        for v in nodes:
            dofs = np.array([u * d + q for u in cols[v, :cnt[v]] for q in range(d)])
            for k in range(d):
                a, b = rp[v * d + k], rp[v * d + k + 1]
                assert np.array_equal(g["cols"][a:b], dofs)
                assert vals[v, k, :b - a].tobytes() == want[a:b].tobytes()
