"""GPU: the symbolic phase's own device primitives (csrc/prims.cu) against numpy.

The reference builds its pattern with std::sort / std::unique per row and a running sum
(pattern.cpp:24-108); the GPU symbolic phase uses a stable LSD radix sort and an exclusive
scan written for this library. Both are integer work: bit-exact.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 31, 32, 33, 2047, 2048, 2049, 4096 * 3 + 5, 1 << 20, (1 << 22) + 12345]


@pytest.fixture(scope="module")
def fea():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2012_00585_b200 as fea
    return fea


@pytest.mark.parametrize("n", SIZES)
def test_exclusive_sum_matches_numpy(fea, n):
    import torch
    rng = np.random.default_rng(n)
    x = rng.integers(-5, 1 << 33, size=n, dtype=np.int64)  # totals far beyond 2^32
    want = np.concatenate(([0], np.cumsum(x)[:-1])) if n else np.zeros(0, np.int64)
    d = torch.from_numpy(x).cuda()
    got = fea.exclusive_sum(d)
    assert np.array_equal(got.cpu().numpy(), want)
    assert np.array_equal(d.cpu().numpy(), x)  # input intact
    got2 = fea.exclusive_sum(d, out=d)  # in place
    assert np.array_equal(got2.cpu().numpy(), want)


@pytest.mark.parametrize("bits", [(0, 32), (0, 1), (0, 9), (0, 17), (0, 25), (4, 20), (0, 0)])
@pytest.mark.parametrize("n", [0, 1, 33, 2049, 100_003, (1 << 21) + 77])
def test_sort_pairs_stable_matches_numpy(fea, n, bits):
    import torch
    b0, b1 = bits
    rng = np.random.default_rng(n * 37 + b1)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    if n > 10:
        keys[: n // 3] = keys[0]  # long runs of equal keys: stability matters
    vals = np.arange(n, dtype=np.int32)
    digit = (keys.astype(np.uint64) >> np.uint64(b0)) & np.uint64((1 << (b1 - b0)) - 1)
    order = np.argsort(digit, kind="stable")
    dk = torch.from_numpy(keys.view(np.int32)).cuda()
    dv = torch.from_numpy(vals).cuda()
    ko, vo = fea.sort_pairs(dk, dv, b0, b1)
    assert np.array_equal(vo.cpu().numpy(), vals[order])
    assert np.array_equal(ko.cpu().numpy().view(np.uint32), keys[order])
    assert np.array_equal(dk.cpu().numpy().view(np.uint32), keys)  # inputs intact
    assert np.array_equal(dv.cpu().numpy(), vals)


def test_sort_pairs_sorted_and_reversed_inputs(fea):
    import torch
    n = 300_000
    for keys in (np.arange(n, dtype=np.uint32), np.arange(n, dtype=np.uint32)[::-1].copy(),
                 np.zeros(n, np.uint32), np.full(n, 0xFFFFFFFF, np.uint32)):
        vals = np.arange(n, dtype=np.int32)
        ko, vo = fea.sort_pairs(torch.from_numpy(keys.view(np.int32)).cuda(), torch.from_numpy(vals).cuda())
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(vo.cpu().numpy(), vals[order])
        assert np.array_equal(ko.cpu().numpy().view(np.uint32), keys[order])
