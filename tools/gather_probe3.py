"""Bare memory pattern of the sorted route on the REAL cfg2 incidence order vs random ids
(no arithmetic): per node read its row blocks, write its values block."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea
from paper_2012_00585_b200 import meshgen as M
from torch.utils.cpp_extension import load_inline

src = r'''
#include <cuda_runtime.h>
__global__ void pattern(const double* __restrict__ K, const int* __restrict__ adj, const long* __restrict__ adj_ptr,
                        const long* __restrict__ nptr, long n_nodes, double* __restrict__ out, int write, int dm) {
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long v = warp; v < n_nodes; v += nw) {
        long b0 = adj_ptr[v], b1 = adj_ptr[v + 1];
        double s = 0;
        for (long c = b0; c < b1; ++c) {
            const double2* src = reinterpret_cast<const double2*>(K + (long)adj[c] * dm);
            double2 a = __ldcs(src + lane); s += a.x + a.y;
            if (lane < dm / 2 - 32) { double2 b = __ldcs(src + 32 + lane); s += b.x + b.y; }
        }
        long vb = 9 * nptr[v]; long blk = 9 * (nptr[v + 1] - nptr[v]);
        if (write) for (long i = lane; i < blk; i += 32) __stcs(out + vb + i, s + i);
        else if (s == 1.2345) out[0] = s;
    }
}
void run(torch::Tensor K, torch::Tensor adj, torch::Tensor adj_ptr, torch::Tensor nptr, torch::Tensor out, int write, int grid, int bs) {
    pattern<<<grid, bs>>>(K.data_ptr<double>(), adj.data_ptr<int>(), adj_ptr.data_ptr<long>(), nptr.data_ptr<long>(),
                          adj_ptr.numel() - 1, out.data_ptr<double>(), write, 72);
}
'''
mod = load_inline("probe3", cpp_sources="void run(torch::Tensor K, torch::Tensor adj, torch::Tensor adj_ptr, torch::Tensor nptr, torch::Tensor out, int write, int grid, int bs);",
                  cuda_sources=src, functions=["run"], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False)
# build the real cfg2 adjacency on the host (node -> incidences ascending element)
import numpy as np
conn, nn, d = M.config_mesh(2)
E, npe = conn.shape
order = np.argsort(conn.reshape(-1), kind="stable")
adj = order.astype(np.int32)  # incidence index e*npe+a, sorted by node then element
cnt = np.bincount(conn.reshape(-1), minlength=nn)
adj_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
plan = fea.Plan(M.element_dofs(conn, d), nn * d, dofs_per_node=d)
rp, _ = plan.csr()
nptr = (rp[::3] // 9).astype(np.int64)
K = fea.fill_seeded_k(E, 24, 42)
out = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
t_adj = torch.from_numpy(adj).cuda(); t_ptr = torch.from_numpy(adj_ptr).cuda(); t_nptr = torch.from_numpy(nptr).cuda()
rnd = torch.from_numpy(np.random.default_rng(1).integers(0, E * npe, size=len(adj)).astype(np.int32)).cuda()
for name, a in (("real", t_adj), ("random", rnd)):
    for write in (0, 1):
        for grid, bs in ((148 * 16, 256), (148 * 32, 128), (148 * 8, 256)):
            mod.run(K, a, t_ptr, t_nptr, out, write, grid, bs)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): mod.run(K, a, t_ptr, t_nptr, out, write, grid, bs)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"{name:7s} write={write} grid={grid} bs={bs}: {ms:.3f} ms")
