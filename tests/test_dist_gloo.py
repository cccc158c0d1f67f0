"""CPU, world_size 2 over gloo: the row-partitioned path end to end on the host side.

Each rank owns a contiguous node range, keeps the elements touching it, builds its row block
(here with the CPU oracle standing in for the device plan, whose block parity is covered by
tests/test_gpu_parity.py::test_row_partition_blocks_concatenate), then the blocks are gathered
to rank 0 with dist.gather_row_blocks and must equal the whole-matrix assembly bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist

    import oracle
    from paper_2012_00585_b200 import dist, meshgen as M
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = 3
        conn, nn = M.hex8_box(3, 3, 4)
        conn = M.permute_elements(conn, 7)
        ed = M.element_dofs(conn, d)
        K = oracle.fill_k(42, conn.shape[0], ed.shape[1])
        lo, hi = dist.owned_node_range(nn, world, rank)
        kept = dist.kept_elements(conn, lo, hi)
        # local block: rows of owned nodes, from the kept elements only
        P = oracle.Pattern.build(conn[kept], nn, d)
        rp, _ = P.arrays()
        full_local = P.assemble_sequential(ed[kept], K[kept])
        block = full_local[rp[lo * d]:rp[hi * d]]
        got = dist.gather_row_blocks(torch.from_numpy(block), root=0)
        # the owned block's CSR / CRAC arrays (rows rebased, global columns), as the plan returns them
        brp = rp[lo * d:hi * d + 1] - rp[lo * d]
        _, cs_all = P.arrays()
        bcs = cs_all[rp[lo * d]:rp[hi * d]]
        Pb = oracle.Pattern.from_arrays(brp, bcs)
        bcp, bca = Pb.crac()
        full = dist.gather_csr_blocks(torch.from_numpy(brp), torch.from_numpy(bcs), torch.from_numpy(block))
        crac = dist.gather_crac_blocks(torch.from_numpy(bcp), torch.from_numpy(bca))
        if rank == 0:
            Pf = oracle.Pattern.build(conn, nn, d)
            want = Pf.assemble_sequential(ed, K)
            frp, fcs = Pf.arrays()
            fcp, fca = Pf.crac()
            ok = got.numpy().tobytes() == want.tobytes()
            ok &= np.array_equal(full[0].numpy(), frp) and np.array_equal(full[1].numpy(), fcs)
            ok &= full[2].numpy().tobytes() == want.tobytes()
            ok &= np.array_equal(crac[0].numpy(), fcp) and np.array_equal(crac[1].numpy(), fca)
            q.put(bool(ok))
    finally:
        tdist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_row_blocks_gather_to_full_matrix():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
