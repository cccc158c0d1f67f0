// y = A x on the assembled matrix — the consumer the paper names as the payoff of CRAC's
// alignment. Three layouts of the same values array
// (row-major, ascending columns; identical for CSR and CRAC, verify.cpp:30-31):
//   * CSR   (row_ptr, int64 cols)                  index bytes: 8 per entry
//   * CRAC  (row_ptr in col_align units, (col_start, values_pos) pairs, final (0, nnz) pair,
//            formats.cpp:21-41)                     index bytes: 16 per run (~0.22 runs/entry on hex8 d=3)
//   * node blocks (the plan's node-level pattern)   index bytes: 4 per d x d block
// All are HBM-bound streaming kernels: one warp per row (CSR/CRAC) or per node (blocks);
// values are read once with streaming loads, x is L2-resident, y written once.
#include "internal.cuh"

namespace feagpu {
extern thread_local std::string g_err;
}

using namespace feagpu;

namespace {

constexpr int kThreads = 256;

unsigned grid_rows(int64_t rows_per_warp_units) {
    int64_t b = (rows_per_warp_units * 32 + kThreads - 1) / kThreads;
    if (b < 1) b = 1;
    if (b > 148 * 64) b = 148 * 64;
    return static_cast<unsigned>(b);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// sum over aligned groups of G lanes (G = 8, 16, 32)
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// lanes per row for rows of `avg` entries on average: a warp per row leaves half its lanes idle
// on tet4 / quad4 d = 1 rows (15 / 9 entries)
inline int group_for(double avg) { return avg <= 10.0 ? 8 : avg <= 24.0 ? 16 : 32; }

// (three entries per lane in flight: values and column loads first, then the x gathers — a row
// of cfg2 has 81 entries, one pass)
// (three entries per lane in flight: values and column loads first, then the x gathers — a row
// of cfg2 has 81 entries, one pass: cfg2 0.231 -> 0.198 ms, cfg4 1.64 -> 1.30 ms)
__global__ void k_spmv_csr(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ cols,
                           const double* __restrict__ values, int64_t n_rows,
                           const double* __restrict__ x, double* __restrict__ y) {
    constexpr int U = 3;
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n_rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        const int64_t i1 = row_ptr[r + 1];
        for (int64_t i0 = row_ptr[r] + lane; i0 < i1; i0 += 32 * U) {
            double a[U];
            int64_t c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + 32 * u;
                a[u] = i < i1 ? __ldcs(values + i) : 0.0;
                c[u] = i < i1 ? __ldcs(cols + i) : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) s += a[u] * __ldg(x + c[u]);
        }
        s = warp_sum(s);
        if (lane == 0) y[r] = s;
    }
}

// CRAC: lane j holds run j of the row (up to 32 runs per pass); entry i of the row finds its
// run (the last run whose values position is <= i) by a 5-step shuffle binary search — the runs
// are ascending in values position — and reads x at col_start + (i - values_pos). On the GPU
// this is instruction-bound (the aligned-run saving targets CPU SIMD slices); the node-block
// layout below realizes the same aligned-column saving with one index per d x d block.
__global__ void k_spmv_crac(const int64_t* __restrict__ crac_ptr, const int64_t* __restrict__ col_align,
                            const double* __restrict__ values, int64_t n_rows,
                            const double* __restrict__ x, double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n_rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a0 = crac_ptr[r], a1 = crac_ptr[r + 1];
        double s = 0.0;
        for (int64_t j0 = a0; j0 < a1; j0 += 64) {  // 32 runs (pairs) per pass
            const int64_t j = j0 + 2 * lane;
            const bool has = j < a1;
            const int64_t cs = has ? col_align[j] : 0;
            const int64_t vs = has ? col_align[j + 1] : INT64_MAX;
            const int nr = __popc(__ballot_sync(0xffffffffu, has));
            const int64_t v_begin = __shfl_sync(0xffffffffu, vs, 0);
            const int64_t v_end = col_align[j0 + 2 * nr + 1];  // next pair's position (or final pair)
            for (int64_t i0 = v_begin; i0 < v_end; i0 += 32) {
                const int64_t i = i0 + lane;
                int k = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = k + step;
                    const int64_t vc = __shfl_sync(0xffffffffu, vs, cand & 31);
                    if (cand < nr && vc <= i) k = cand;
                }
                const int64_t rcs = __shfl_sync(0xffffffffu, cs, k);
                const int64_t rvs = __shfl_sync(0xffffffffu, vs, k);
                if (i < v_end) s += __ldcs(values + i) * __ldg(x + rcs + (i - rvs));
            }
        }
        s = warp_sum(s);
        if (lane == 0) y[r] = s;
    }
}

// Node blocks: the d rows of node v share its neighbour node list; block p covers columns
// ncol[p]*d .. ncol[p]*d+d-1. Warp per node; each lane takes columns q of the block and
// accumulates all d rows at once, so every x element and column index is loaded once.
template <int D, int G>
__global__ void k_spmv_nodes(const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol,
                             int64_t n_own, const double* __restrict__ values,
                             const double* __restrict__ x, double* __restrict__ y) {
    // G lanes per node (G < 32 for short rows: a warp per node leaves half its lanes idle on
    // tet4 / quad4 d = 1 rows of 15 / 9 columns); a warp's groups iterate together
    const int gl = threadIdx.x & (G - 1);
    const int64_t stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * (32 / G);
    for (int64_t v0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (32 / G); v0 < n_own; v0 += stride) {
        const int64_t v = v0 + (threadIdx.x & 31) / G;
        const bool on = v < n_own;
        const int64_t c0 = on ? nptr[v] : 0;
        const int cnt = on ? static_cast<int>(nptr[v + 1] - c0) : 0;
        const int rowlen = D * cnt;
        const double* blk = values + static_cast<int64_t>(D) * D * c0;
        double s[D];
#pragma unroll
        for (int ki = 0; ki < D; ++ki) s[ki] = 0.0;
        // U column groups per lane in flight (a hex8 node row has <= 81 columns: one pass): the
        // values loads do not wait for the column -> x chain
        constexpr int U = G == 32 ? 3 : 2;
        for (int q0 = gl; q0 < rowlen; q0 += G * U) {
            double a[U][D], xv[U];
            int col[U], kj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + G * u;
                const bool ok = q < rowlen;
                const int p = q / D;
                kj[u] = q - p * D;
                col[u] = ok ? __ldg(ncol + c0 + p) : 0;
#pragma unroll
                for (int ki = 0; ki < D; ++ki) a[u][ki] = ok ? __ldcs(blk + ki * rowlen + q) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = __ldg(x + static_cast<int64_t>(col[u]) * D + kj[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int ki = 0; ki < D; ++ki) s[ki] += a[u][ki] * xv[u];
        }
#pragma unroll
        for (int ki = 0; ki < D; ++ki) {
            const double t = group_sum<G>(s[ki]);
            if (gl == 0 && on) y[v * D + ki] = t;
        }
    }
}

template <class F>
fea_status guarded_s(F&& f) {
    try {
        g_err.clear();
        f();
        return FEA_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FEA_ERR_INVALID;
    }
}

}  // namespace

extern "C" {

fea_status fea_spmv_csr(const int64_t* row_ptr, const int64_t* cols, const double* values, int64_t n_rows,
                        const double* x, double* y, void* stream) {
    return guarded_s([&] {
        FEA_REQUIRE(n_rows >= 0 && (n_rows == 0 || (row_ptr && x && y)), FEA_ERR_INVALID, "bad arguments");
        if (n_rows == 0) return;
        k_spmv_csr<<<grid_rows(n_rows), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(row_ptr, cols, values,
                                                                                       n_rows, x, y);
        FEA_CK(cudaGetLastError());
    });
}

fea_status fea_spmv_crac(const int64_t* crac_ptr, const int64_t* col_align, const double* values,
                         int64_t n_rows, const double* x, double* y, void* stream) {
    return guarded_s([&] {
        FEA_REQUIRE(n_rows >= 0 && (n_rows == 0 || (crac_ptr && col_align && x && y)), FEA_ERR_INVALID,
                    "bad arguments");
        if (n_rows == 0) return;
        k_spmv_crac<<<grid_rows(n_rows), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
            crac_ptr, col_align, values, n_rows, x, y);
        FEA_CK(cudaGetLastError());
    });
}

fea_status fea_plan_spmv(const fea_plan* p, const double* values, const double* x, double* y, void* stream) {
    return guarded_s([&] {
        FEA_REQUIRE(p && (p->n_own == 0 || (values && x && y)), FEA_ERR_INVALID, "bad arguments");
        if (p->n_own == 0) return;
        DeviceScope ds(p->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int64_t* np = p->nptr.as<int64_t>();
        const int32_t* nc = p->ncol.as<int32_t>();
        const int gsz = group_for(static_cast<double>(p->d) * static_cast<double>(p->nnz_nodes) /
                                  static_cast<double>(p->n_own));
        const unsigned g = grid_rows((p->n_own * gsz + 31) / 32);
        auto launch = [&](auto k8, auto k16, auto k32) {
            if (gsz == 8) k8<<<g, kThreads, 0, s>>>(np, nc, p->n_own, values, x, y);
            else if (gsz == 16) k16<<<g, kThreads, 0, s>>>(np, nc, p->n_own, values, x, y);
            else k32<<<g, kThreads, 0, s>>>(np, nc, p->n_own, values, x, y);
        };
        switch (p->d) {
            case 1: launch(k_spmv_nodes<1, 8>, k_spmv_nodes<1, 16>, k_spmv_nodes<1, 32>); break;
            case 2: launch(k_spmv_nodes<2, 8>, k_spmv_nodes<2, 16>, k_spmv_nodes<2, 32>); break;
            case 3: launch(k_spmv_nodes<3, 8>, k_spmv_nodes<3, 16>, k_spmv_nodes<3, 32>); break;
            case 4: launch(k_spmv_nodes<4, 8>, k_spmv_nodes<4, 16>, k_spmv_nodes<4, 32>); break;
            default: throw Error(FEA_ERR_INVALID, "fea_plan_spmv supports 1 <= d <= 4");
        }
        FEA_CK(cudaGetLastError());
    });
}

}  // extern "C"
