"""Bare memory pattern of the d = 1 sorted route on the REAL cfg3 traversal (no shared-memory
accumulator, no position decode): per node read the K rows of its incidences (ascending element
id, nodes in the plan's traversal order = sorted by lowest incident element) and write its
values block. Sets the practical floor of this access pattern for k_gather_d1 / k_gather_d1r.

  python tools/gather_probe_d1.py
"""
import sys
from pathlib import Path

import numpy as np
import torch
from torch.utils.cpp_extension import load_inline

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

src = r'''
#include <cuda_runtime.h>
// G lanes per node, lane reads 32/G bytes of each 32 B row; U rows in flight per lane
template <int G, int U>
__global__ void probe(const double* __restrict__ K, const int* __restrict__ rec, const long* __restrict__ tptr,
                      const long* __restrict__ vstart, const int* __restrict__ vlen, long n_nodes,
                      double* __restrict__ out, const int* __restrict__ hi, long la) {
    const long grp = (blockIdx.x * (long)blockDim.x + threadIdx.x) / G;
    const int gl = threadIdx.x % G;
    if (la > 0 && threadIdx.x == 0) {  // L2 prefetch frontier: rows first needed la nodes ahead
        const long per = blockDim.x / G;
        const long ta = blockIdx.x * per + la - 1, tb = min(ta + per, n_nodes - 1);
        if (tb > ta) {
            const long lo = (long)hi[ta] * 32 + 32, h = (long)hi[tb] * 32 + 32;
            for (long b = lo; b < h; b += 65536) {
                const unsigned sz = (unsigned)min(h - b, 65536L);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)K + b), "r"(sz) : "memory");
            }
        }
    }
    if (grp >= n_nodes) return;
    const long a0 = tptr[grp], a1 = tptr[grp + 1];
    double s = 0;
    for (long c = a0; c < a1; c += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = 0;
            if (c + u < a1) {
                const int e = rec[c + u];
                if (G == 4) v[u] = __ldcg(K + (long)e * 4 + gl);
                else { double2 x = __ldcg(reinterpret_cast<const double2*>(K + (long)e * 4) + gl); v[u] = x.x + x.y; }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u];
    }
    const long vb = vstart[grp];
    for (int i = gl; i < vlen[grp]; i += G) __stcs(out + vb + i, s + i);
}
void run(torch::Tensor K, torch::Tensor rec, torch::Tensor tptr, torch::Tensor vs, torch::Tensor vl, torch::Tensor out,
         int g, int u, int bs, torch::Tensor hi, long la) {
    long n = vl.numel();
    long threads = n * g;
    int grid = (threads + bs - 1) / bs;
    auto args = [&](auto kern) { kern<<<grid, bs>>>(K.data_ptr<double>(), rec.data_ptr<int>(), tptr.data_ptr<long>(),
        vs.data_ptr<long>(), vl.data_ptr<int>(), n, out.data_ptr<double>(), hi.data_ptr<int>(), la); };
    if (g == 4 && u == 4) args(probe<4, 4>);
    if (g == 4 && u == 8) args(probe<4, 8>);
    if (g == 4 && u == 24) args(probe<4, 24>);
    if (g == 2 && u == 4) args(probe<2, 4>);
    if (g == 2 && u == 8) args(probe<2, 8>);
    if (g == 2 && u == 24) args(probe<2, 24>);
}
'''
mod = load_inline("probe_d1", cpp_sources="void run(torch::Tensor K, torch::Tensor rec, torch::Tensor tptr, torch::Tensor vs, torch::Tensor vl, torch::Tensor out, int g, int u, int bs, torch::Tensor hi, long la);",
                  cuda_sources=src, functions=["run"],
                  extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False)

conn, nn, d = M.config_mesh(3)
E, npe = conn.shape
flat = conn.reshape(-1)
inc = np.argsort(flat, kind="stable").astype(np.int32)          # incidences by node, ascending element
cnt = np.bincount(flat, minlength=nn)
ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
lowest = inc[ptr[:-1]] // npe                                     # lowest incident element per node
trav = np.argsort(lowest, kind="stable")                          # the plan's traversal order
tcnt = cnt[trav]
tptr = np.concatenate([[0], np.cumsum(tcnt)]).astype(np.int64)
# vectorised gather of the records in traversal order
starts = np.repeat(ptr[trav], tcnt)
offs = np.arange(tptr[-1]) - np.repeat(tptr[:-1], tcnt)
rec = inc[starts + offs].astype(np.int32)
plan = fea.Plan(M.element_dofs(conn, d), nn * d, dofs_per_node=d)
rp, _ = plan.csr()
vs = rp[:-1][trav].astype(np.int64)
vl = np.diff(rp)[trav].astype(np.int32)
K = fea.fill_seeded_k(E, 4, 42)
out = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
T = [torch.from_numpy(x).cuda() for x in (rec, tptr, vs, vl)]
last = rec[np.maximum(tptr[1:] - 1, 0)]                          # highest K row per traversal node
hi = torch.from_numpy(np.maximum.accumulate(last).astype(np.int32)).cuda()
alg = 8 * E * 16 + 8 * plan.nnz + 4 * E * npe
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for g, u, bs, la in [(4, 4, 128, 0), (4, 4, 256, 0), (2, 8, 128, 0), (4, 4, 128, 2048), (4, 4, 128, 8192),
                     (4, 4, 128, 32768), (4, 4, 128, 131072), (4, 4, 256, 8192), (4, 4, 256, 32768)]:
            mod.run(K, *T, out, g, u, bs, hi, la)
            ms = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                mod.run(K, *T, out, g, u, bs, hi, la)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = float(np.mean(ms))
            print(f"G={g} U={u:2d} bs={bs} prefetch-ahead={la}: {t:.3f} ms  ({alg / t / 1e6:.0f} GB/s algorithmic)", flush=True)
