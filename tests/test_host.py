"""CPU: host-side logic (synthetic meshes, row partitioning, bench workload bookkeeping)."""
import numpy as np
import pytest

from paper_2012_00585_b200 import dist, meshgen as M


@pytest.mark.parametrize("mesh,n", [("quad4", 4), ("hex8", 3), ("tet4", 2), ("hex27", 2)])
def test_mesh_shapes_and_conformity(mesh, n):
    conn, nn = M.make_mesh(mesh, n)
    npe = {"quad4": 4, "hex8": 8, "tet4": 4, "hex27": 27}[mesh]
    E = {"quad4": n * n, "hex8": n ** 3, "tet4": 6 * n ** 3, "hex27": n ** 3}[mesh]
    assert conn.shape == (E, npe)
    assert conn.min() == 0 and conn.max() == nn - 1
    for e in range(E):
        assert len(set(conn[e])) == npe
    assert len(np.unique(conn)) == nn  # every node used


def test_permutations_are_bijections():
    p = M.hash_permutation(1000, 7)
    assert np.array_equal(np.sort(p), np.arange(1000))
    assert not np.array_equal(p, np.arange(1000))
    assert np.array_equal(p, M.hash_permutation(1000, 7))
    conn, nn = M.hex8_structured(3)
    pe = M.permute_elements(conn, 7)
    assert sorted(map(tuple, pe)) == sorted(map(tuple, conn))
    pn = M.permute_nodes(conn, nn, 7)
    assert len(np.unique(pn)) == nn


def test_element_dofs_node_contiguous():
    conn, _ = M.hex8_structured(2)
    ed = M.element_dofs(conn, 3)
    assert ed.shape == (8, 24)
    assert np.array_equal(ed[:, 0::3] // 3, conn) and np.all(ed[:, 1::3] == ed[:, 0::3] + 1)


def test_hex8_box_matches_cube():
    a, na = M.hex8_box(3, 3, 3)
    b, nb = M.hex8_structured(3)
    assert na == nb and np.array_equal(a, b)


def test_owned_ranges_partition_rows():
    for world in (1, 2, 3, 8):
        ranges = [dist.owned_row_range(1001, 3, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 3003
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert all(lo % 3 == 0 and hi % 3 == 0 for lo, hi in ranges)
    w = np.ones(100)
    w[:10] = 50
    lo, hi = dist.owned_node_range(100, 2, 0, weights=w)
    assert lo == 0 and hi < 50


def test_kept_elements_and_halo():
    conn, nn = M.hex8_box(4, 4, 8)
    lo, hi = dist.owned_node_range(nn, 2, 0)
    kept = dist.kept_elements(conn, lo, hi)
    assert np.all(np.any((conn[kept] >= lo) & (conn[kept] < hi), axis=1))
    others = np.setdiff1d(np.arange(conn.shape[0]), kept)
    assert not np.any((conn[others] >= lo) & (conn[others] < hi))
    assert 0 < dist.redundant_fraction(conn, nn, 2) < 0.3


def test_bench_rank_node_ranges_cover_mesh_and_balance():
    """bench.py --gpus N: contiguous node ranges covering the config-5 mesh (here at n=32),
    cut at incidence quantiles: per-rank incidence counts within 2 % of each other."""
    import bench
    conn, nn = M.hex8_structured(32)
    w = np.bincount(conn.ravel(), minlength=nn)
    for N in (1, 2, 4, 8):
        ranges = [bench.rank_nodes(conn, nn, N, r) for r in range(N)]
        assert ranges[0][0] == 0 and ranges[-1][1] == nn
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        loads = [w[lo:hi].sum() for lo, hi in ranges]
        assert max(loads) <= 1.02 * min(loads)
