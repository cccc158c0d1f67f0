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
                      double* __restrict__ out, const int* __restrict__ hi, long la, int wmode) {
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
    // wmode 0: the real values rows (node-id order: random 120 B rows); 1: no writes (kept live);
    // 2: the same rows written in traversal order (sequential)
    const long vb = wmode == 2 ? grp * 16 : vstart[grp];
    if (wmode == 1) { if (s == 1.2345e300) out[0] = s; return; }
    for (int i = gl; i < vlen[grp]; i += G) __stcs(out + vb + i, s + i);
}
// 8-byte records {entry, slot word} and a shared-memory fold (slot = byte gl of the word mod
// row length): the kernel's record width and accumulator traffic on the same traversal
template <int U, bool SMEM, bool LDG>
__global__ void probe_fold(const double* __restrict__ K, const int2* __restrict__ rec, const long* __restrict__ tptr,
                           const long* __restrict__ vstart, const int* __restrict__ vlen, long n_nodes,
                           double* __restrict__ out) {
    __shared__ double acc[64 * 19];
    const int grp = threadIdx.x >> 2, gl = threadIdx.x & 3;
    const long node = blockIdx.x * 64L + grp;
    long a0 = 0, a1 = 0; int rl = 1;
    if (node < n_nodes) { a0 = tptr[node]; a1 = tptr[node + 1]; rl = vlen[node]; }
    double* A = acc + grp * 19;
    for (int i = gl; i < rl; i += 4) A[i] = 0;
    double s = 0;
    for (long c = a0; c < a1; c += U) {
        int2 r[U]; double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = c + u < a1 ? (LDG ? __ldg(rec + c + u) : __ldcs(rec + c + u)) : make_int2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = c + u < a1 ? __ldcg(K + (long)r[u].x * 4 + gl) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (SMEM) { if (c + u < a1) { const int q = ((unsigned)r[u].y >> (8 * gl) & 0xff) % rl; A[q] += v[u]; } __syncwarp(); }
            else s += v[u] + r[u].y;
        }
    }
    __syncwarp();
    if (node < n_nodes) { const long vb = vstart[node]; for (int i = gl; i < rl; i += 4) __stcs(out + vb + i, SMEM ? A[i] : s + i); }
}
void run_fold(torch::Tensor K, torch::Tensor rec2, torch::Tensor tptr, torch::Tensor vs, torch::Tensor vl, torch::Tensor out, int smem) {
    long n = vl.numel();
    int grid = (n + 63) / 64;
    if (smem == 2) probe_fold<4, false, true><<<grid, 256>>>(K.data_ptr<double>(), (const int2*)rec2.data_ptr<int>(), tptr.data_ptr<long>(), vs.data_ptr<long>(), vl.data_ptr<int>(), n, out.data_ptr<double>());
    else if (smem == 3) probe_fold<4, true, true><<<grid, 256>>>(K.data_ptr<double>(), (const int2*)rec2.data_ptr<int>(), tptr.data_ptr<long>(), vs.data_ptr<long>(), vl.data_ptr<int>(), n, out.data_ptr<double>());
    else if (smem) probe_fold<4, true, false><<<grid, 256>>>(K.data_ptr<double>(), (const int2*)rec2.data_ptr<int>(), tptr.data_ptr<long>(), vs.data_ptr<long>(), vl.data_ptr<int>(), n, out.data_ptr<double>());
    else probe_fold<4, false, false><<<grid, 256>>>(K.data_ptr<double>(), (const int2*)rec2.data_ptr<int>(), tptr.data_ptr<long>(), vs.data_ptr<long>(), vl.data_ptr<int>(), n, out.data_ptr<double>());
}
void run(torch::Tensor K, torch::Tensor rec, torch::Tensor tptr, torch::Tensor vs, torch::Tensor vl, torch::Tensor out,
         int g, int u, int bs, torch::Tensor hi, long la, int wmode) {
    long n = vl.numel();
    long threads = n * g;
    int grid = (threads + bs - 1) / bs;
    auto args = [&](auto kern) { kern<<<grid, bs>>>(K.data_ptr<double>(), rec.data_ptr<int>(), tptr.data_ptr<long>(),
        vs.data_ptr<long>(), vl.data_ptr<int>(), n, out.data_ptr<double>(), hi.data_ptr<int>(), la, wmode); };
    if (g == 4 && u == 4) args(probe<4, 4>);
    if (g == 4 && u == 8) args(probe<4, 8>);
    if (g == 4 && u == 24) args(probe<4, 24>);
    if (g == 2 && u == 4) args(probe<2, 4>);
    if (g == 2 && u == 8) args(probe<2, 8>);
    if (g == 2 && u == 24) args(probe<2, 24>);
}
'''
mod = load_inline("probe_d1", cpp_sources="void run(torch::Tensor K, torch::Tensor rec, torch::Tensor tptr, torch::Tensor vs, torch::Tensor vl, torch::Tensor out, int g, int u, int bs, torch::Tensor hi, long la, int wmode); void run_fold(torch::Tensor K, torch::Tensor rec2, torch::Tensor tptr, torch::Tensor vs, torch::Tensor vl, torch::Tensor out, int smem);",
                  cuda_sources=src, functions=["run", "run_fold"],
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
out = torch.empty(max(plan.nnz, 16 * nn + 16), dtype=torch.float64, device="cuda")
T = [torch.from_numpy(x).cuda() for x in (rec, tptr, vs, vl)]
last = rec[np.maximum(tptr[1:] - 1, 0)]                          # highest K row per traversal node
hi = torch.from_numpy(np.maximum.accumulate(last).astype(np.int32)).cuda()
words = (rec.astype(np.uint64) * np.uint64(2654435761) >> np.uint64(7)).astype(np.uint32).view(np.int32)
rec2 = torch.from_numpy(np.stack([rec, words], axis=1).reshape(-1).copy()).cuda()
alg = 8 * E * 16 + 8 * plan.nnz + 4 * E * npe
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for g, u, bs, la, wm in [(4, 4, 256, 0, 0), (4, 4, 256, 0, 1), (4, 4, 256, 0, 2), (2, 8, 128, 0, 0), (4, 4, 256, 8192, 0)]:
            mod.run(K, *T, out, g, u, bs, hi, la, wm)
            ms = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                mod.run(K, *T, out, g, u, bs, hi, la, wm)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = float(np.mean(ms))
            print(f"G={g} U={u:2d} bs={bs} prefetch-ahead={la} writes={("rows", "none", "sequential")[wm]}: {t:.3f} ms  ({alg / t / 1e6:.0f} GB/s algorithmic)", flush=True)

for smem in (0, 1, 2, 3):
    mod.run_fold(K, rec2, T[1], T[2], T[3], out, smem)
    ms = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mod.run_fold(K, rec2, T[1], T[2], T[3], out, smem)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.mean(ms))
    print(f"8-byte records, U=4, {'shared-memory fold' if smem in (1, 3) else 'register sum'}, records {'ld.global.nc' if smem >= 2 else 'ld.global.cs'}: {t:.3f} ms  ({alg / t / 1e6:.0f} GB/s algorithmic)", flush=True)
