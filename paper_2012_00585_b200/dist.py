"""Row-partitioned multi-GPU assembly: ownership, element filtering, optional row-block gather.

SURVEY.md §8e: each rank owns a contiguous range of node rows; it keeps the elements with at
least one node in its range (the plan does that on the device), assembles its row block with
no collective, and the row blocks can optionally be gathered to one rank over NCCL. There is
no reference counterpart (the reference is shared-memory only); this module is the
host side of that B200 extension and works with any torch.distributed backend (NCCL on GPUs,
gloo on CPU for the tests).
"""
from __future__ import annotations

import numpy as np


def owned_node_range(n_nodes: int, world: int, rank: int, weights=None):
    """Contiguous node range of `rank`: equal node counts, or balanced by `weights`
    (e.g. node-level NNZ) at the weight quantiles."""
    if weights is None:
        return n_nodes * rank // world, n_nodes * (rank + 1) // world
    c = np.concatenate([[0], np.cumsum(np.asarray(weights, dtype=np.float64))])
    total = c[-1]
    cut = lambda r: int(np.searchsorted(c, total * r / world, side="left"))  # noqa: E731
    lo = 0 if rank == 0 else cut(rank)
    hi = n_nodes if rank == world - 1 else cut(rank + 1)
    return lo, hi


def owned_row_range(n_nodes: int, d: int, world: int, rank: int, weights=None):
    lo, hi = owned_node_range(n_nodes, world, rank, weights)
    return lo * d, hi * d


def kept_elements(conn: np.ndarray, node_lo: int, node_hi: int) -> np.ndarray:
    """Ids (ascending) of the elements with at least one node in [node_lo, node_hi) — the
    host mirror of the plan's device-side element filter."""
    own = (conn >= node_lo) & (conn < node_hi)
    return np.nonzero(own.any(axis=1))[0].astype(np.int64)


def redundant_fraction(conn: np.ndarray, n_nodes: int, world: int) -> float:
    """Extra element work of row partitioning: sum of kept elements over ranks / E - 1."""
    total = 0
    for r in range(world):
        lo, hi = owned_node_range(n_nodes, world, r)
        total += len(kept_elements(conn, lo, hi))
    return total / conn.shape[0] - 1.0


def gather_row_blocks(values_local, root: int = 0, group=None):
    """Gather every rank's row block of values (1-D, any length) to `root`, concatenated in
    rank order (= global row order for contiguous ownership). Returns the full values array on
    `root` and None elsewhere. Lengths are exchanged first, so blocks may differ in size."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([values_local.numel()], dtype=torch.int64, device=values_local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    buf = torch.zeros(mx, dtype=values_local.dtype, device=values_local.device)
    buf[: values_local.numel()] = values_local
    out = [torch.empty_like(buf) for _ in range(world)] if rank == root else None
    dist.gather(buf, out, dst=root, group=group)
    if rank != root:
        return None
    return torch.cat([o[:s] for o, s in zip(out, sizes)])


class PeerValues:
    """Fused assembly + gather over peer memory: the root allocates the GLOBAL values array,
    exports it (CUDA IPC, fea_ipc_export) and every rank maps it (fea_ipc_open); rank r's row
    block starts at the sum of the NNZ of the ranks before it (contiguous ownership = global row
    order). Each rank then assembles straight into `ptr` (Plan.assemble_into): the numeric
    kernel's value stores travel over NVLink/NVSwitch while the block is assembled, instead of
    an NCCL gather after the kernel. After every rank's stream has finished and a barrier,
    `full` on the root holds the global values. Collective: every rank constructs it.
    """

    def __init__(self, local_nnz: int, device, root: int = 0, group=None):
        import ctypes
        from ctypes import byref, c_int64, c_void_p

        import torch
        import torch.distributed as dist

        from . import _native as N
        from .assembly import _check
        self._lib = N.lib()
        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        sizes = [None] * world
        dist.all_gather_object(sizes, int(local_nnz), group=group)
        self.offset = int(sum(sizes[: self.rank]))
        self.total = int(sum(sizes))
        self.full = None
        self._base = None
        obj = [None]
        if self.rank == root:
            self.full = torch.zeros(max(self.total, 1), dtype=torch.float64, device=device)
            h = ctypes.create_string_buffer(64)
            off = c_int64()
            _check(self._lib.fea_ipc_export(c_void_p(self.full.data_ptr()), h, byref(off)))
            obj = [(h.raw, off.value)]
        dist.broadcast_object_list(obj, src=root, group=group)
        if self.rank == root:
            base = self.full.data_ptr()
        else:
            handle, off = obj[0]
            b = c_void_p()
            _check(self._lib.fea_ipc_open(ctypes.create_string_buffer(handle, 64), int(torch.device(device).index or 0),
                                          byref(b)))
            self._base = b
            base = b.value + off
        self.ptr = base + 8 * self.offset  # this rank's row block

    def close(self) -> None:
        if self._base is not None:
            self._lib.fea_ipc_close(self._base)
            self._base = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _gather_1d(t, root, group):
    """Gather a 1-D tensor of any length from every rank to `root` (rank order)."""
    return gather_row_blocks(t, root=root, group=group)


def gather_csr_blocks(row_ptr, cols, values, root: int = 0, group=None):
    """Rebuild the global CSR matrix on `root` from every rank's owned row block
    (row_ptr rebased to 0 per block, global cols). Returns (row_ptr, cols, values) on root."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    rp = _gather_1d(row_ptr[1:].contiguous(), root, group)  # drop each block's leading 0
    cs = _gather_1d(cols, root, group)
    vs = _gather_1d(values, root, group)
    counts = torch.tensor([row_ptr.numel() - 1, values.numel()], dtype=torch.int64, device=row_ptr.device)
    world = dist.get_world_size(group)
    allc = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    if rank != root:
        return None
    out = [torch.zeros(1, dtype=row_ptr.dtype, device=row_ptr.device)]
    pos, base = 0, 0
    for c in allc:
        nr, nz = int(c[0]), int(c[1])
        out.append(rp[pos:pos + nr] + base)
        pos += nr
        base += nz
    return torch.cat(out), cs, vs


def gather_crac_blocks(crac_ptr, col_align, root: int = 0, group=None):
    """Rebuild the global CRAC arrays on `root`: each block's row_ptr (col_align entry units) and
    its (col_start, values_pos) pairs are rebased by the blocks before it; one final (0, nnz)
    pair closes the result (formats.cpp:36-39)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    nr = crac_ptr.numel() - 1
    pairs = col_align[:-2].contiguous()  # drop the block's final pair
    nnz = col_align[-1:].clone()
    meta = torch.tensor([nr, pairs.numel(), int(nnz.item())], dtype=torch.int64, device=crac_ptr.device)
    allm = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(allm, meta, group=group)
    rp = _gather_1d(crac_ptr[1:].contiguous(), root, group)
    pa = _gather_1d(pairs, root, group)
    if rank != root:
        return None
    ptr_out = [torch.zeros(1, dtype=crac_ptr.dtype, device=crac_ptr.device)]
    pair_out = []
    rpos = ppos = 0
    abase = vbase = 0
    for m in allm:
        nrb, npb, nzb = int(m[0]), int(m[1]), int(m[2])
        ptr_out.append(rp[rpos:rpos + nrb] + abase)
        blk = pa[ppos:ppos + npb].clone()
        blk[1::2] += vbase
        pair_out.append(blk)
        rpos += nrb
        ppos += npb
        abase += npb
        vbase += nzb
    pair_out.append(torch.tensor([0, vbase], dtype=col_align.dtype, device=col_align.device))
    return torch.cat(ptr_out), torch.cat(pair_out)
