// Symbolic phase of the B200 FE-assembly library (north-star subsystem 1) and
// the per-element local->global slot map (subsystem 2), plus the plan's C ABI.
//
// Reference behaviour restated (not translated):
//   build_pattern         pattern.cpp:24-108  node->element index, per-node
//                         gather + sort/unique, replicate to the node's d rows
//   count_pattern_runs    pattern.cpp:110-120
//   build_crac_arrays     formats.cpp:21-41
//   CsrBase/CracBase::locate formats.hpp:165-199, :276-290 (external patterns)
//   greedy_colouring      colouring.cpp:24-75
//   find_colour_conflict  colouring.cpp:91-119
//
// B200 layout: everything is stored per NODE (the d rows of a node share one
// column list, pattern.cpp:85-91) and expanded arithmetically:
//   row (v,k) of the owned block starts at  d*d*nptr[v] + k*d*cnt(v)
//   entry (v,k ; u,kj) lives at             row_start + d*pos(v,u) + kj
// so the slot map is one small row-relative position per (element, node a,
// node b) — uint8 when every node row has <= 256 neighbour nodes — instead of
// an int32/int64 slot per element-matrix entry.

#include <chrono>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"
#include "prims.cuh"

namespace feagpu {

thread_local std::string g_err;

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    cudaGetLastError();  // clear sticky-free errors
    const fea_status s = (e == cudaErrorMemoryAllocation) ? FEA_ERR_OOM : FEA_ERR_CUDA;
    throw Error(s, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                       std::to_string(line) + ")");
}

void DevBuf::alloc(size_t n) {
    reset();
    bytes = n;
    FEA_CK(cudaMalloc(&p, n < 256 ? 256 : n));
}

void DevBuf::reset() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

DeviceScope::DeviceScope(int dev) {
    FEA_CK(cudaGetDevice(&prev));
    if (prev != dev) FEA_CK(cudaSetDevice(dev));
}
DeviceScope::~DeviceScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

Knobs read_knobs() {
    auto on = [](const char* n) { return std::getenv(n) != nullptr; };
    auto mod = [](const char* n) {
        const char* e = std::getenv(n);
        return e ? (std::atoi(e) & 15) : -1;
    };
    return Knobs{on("FEA_ATOMIC_LEGACY"), on("FEA_ATOMIC_NO_PATCH"), on("FEA_SLOT_NO_FIXED"), on("FEA_CN_UNPACKED"),
                 on("FEA_CN_NO_RECORDS"), on("FEA_D1_NO_DIRECT"),    on("FEA_D1_NO_VEC"),
                 on("FEA_D1_NO_LANE"),    on("FEA_ATOMIC_NO_STRIP"), on("FEA_PATCH_TICKETS"), on("FEA_PATCH_STATIC"), on("FEA_GATHER_GLOBAL"), on("FEA_D1_REC8"),
                 mod("FEA_D1_ACC_STRIDE_MOD16"), mod("FEA_D1V_ACC_STRIDE_MOD16")};
}

void HostPipe::ensure_events(int n) {
    if (!sin) {
        FEA_CK(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking));
        FEA_CK(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking));
    }
    while (static_cast<int>(ev.size()) < n) {
        cudaEvent_t e = nullptr;
        FEA_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev.push_back(e);
    }
}

HostPipe::~HostPipe() {
    if (sin) cudaStreamSynchronize(sin);
    if (sout) cudaStreamSynchronize(sout);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (sin) cudaStreamDestroy(sin);
    if (sout) cudaStreamDestroy(sout);
}

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kNodeCap = 512;  // candidates sorted in a warp's shared-memory slice

// FEA_PLAN_TRACE: per-stage wall time of the symbolic phase on stderr (synchronises the plan
// stream at every mark; measurement only)
struct StageTrace {
    bool on = std::getenv("FEA_PLAN_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what, cudaStream_t s) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "plan trace: %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

bool is_device_ptr(const void* ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 64) b = 148 * 64;  // grid-stride beyond ~64 CTAs per SM
    return static_cast<unsigned>(b);
}

int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (x >> b) != 0) ++b;
    return b;
}

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------

// Flat DOFs -> node ids, validating range and (for d > 1) the node-contiguous
// layout dof(v,k) = v*d+k (dof_map.hpp:59). flags bit0: layout broken,
// bit1: DOF out of [0, n_rows) (the reference's out_of_range, dof_map.cpp:82-84).
__global__ void k_extract_conn(const int64_t* __restrict__ dofs, int64_t total, int m, int d,
                               int npe, int64_t n_rows, int32_t* __restrict__ conn,
                               unsigned* flags) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t / npe;
        const int a = static_cast<int>(t - e * npe);
        const int64_t* src = dofs + e * m + (int64_t)a * d;
        const int64_t base = src[0];
        unsigned f = 0;
        if (base < 0 || base >= n_rows) f |= 2u;
        if (d > 1) {
            if (base % d != 0) f |= 1u;
            for (int k = 1; k < d; ++k) {
                const int64_t x = src[k];
                if (x != base + k) f |= 1u;
                if (x < 0 || x >= n_rows) f |= 2u;
            }
        }
        // a node repeated inside one element (bit 2): the reference adds both
        // occurrences in order; the gather then keeps a serialised fold
        for (int b = 0; b < a; ++b)
            if (dofs[e * m + (int64_t)b * d] == base) f |= 4u;
        if (f) atomicOr(flags, f);
        conn[t] = static_cast<int32_t>(base / d);
    }
}

__global__ void k_keep_flags(const int32_t* __restrict__ conn, int64_t E, int npe, int64_t nb,
                             int64_t ne, int64_t* __restrict__ keep) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = 0;
        for (int a = 0; a < npe; ++a) {
            const int64_t v = conn[e * npe + a];
            k |= (v >= nb && v < ne) ? 1 : 0;
        }
        keep[e] = k;
    }
}

__global__ void k_scatter_kept(const int64_t* __restrict__ keep, const int64_t* __restrict__ pos,
                               int64_t E, int64_t* __restrict__ elem_id) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        if (keep[e]) elem_id[pos[e]] = e;
}

__global__ void k_iota64(int64_t* x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = i;
}

__global__ void k_krow(const int64_t* __restrict__ elem_id, int64_t E, bool compact,
                       int32_t* __restrict__ krow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x)
        krow[i] = static_cast<int32_t>(compact ? i : elem_id[i]);
}

__global__ void k_gather_conn(const int32_t* __restrict__ conn_all, const int64_t* __restrict__ elem_id,
                              int64_t E, int npe, int32_t* __restrict__ conn) {
    const int64_t total = E * npe;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t le = t / npe;
        conn[t] = conn_all[elem_id[le] * npe + (t - le * npe)];
    }
}

// (node, element) incidences, emitted in ascending element order; the stable
// radix sort by node then leaves each node's list in ascending element id —
// the node->element index of pattern.cpp:32-48.
__global__ void k_emit_incidences(const int32_t* __restrict__ conn_k,
                                  const int32_t* __restrict__ krow, int64_t E, int npe,
                                  int64_t nb, int64_t ne, uint32_t* __restrict__ keys,
                                  int32_t* __restrict__ vals,
                                  unsigned long long* __restrict__ counts) {
    const int64_t total = E * npe;
    const uint32_t sentinel = static_cast<uint32_t>(ne - nb);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t le = t / npe;
        const int a = static_cast<int>(t - le * npe);
        const int64_t kr = krow[le];
        const int64_t v = conn_k[kr * npe + a];
        const bool own = v >= nb && v < ne;
        keys[t] = own ? static_cast<uint32_t>(v - nb) : sentinel;
        vals[t] = static_cast<int32_t>(kr * npe + a);
        if (own) atomicAdd(counts + (v - nb), 1ull);
    }
}

__device__ __forceinline__ int32_t candidate(const int32_t* __restrict__ adj,
                                             const int32_t* __restrict__ conn_k, int64_t b0,
                                             int npe, int64_t i) {
    const int64_t k = i / npe;
    const int b = static_cast<int>(i - k * npe);
    const int32_t entry = adj[b0 + k];
    return conn_k[(int64_t)(entry - entry % npe) + b];
}

// Warp-level bitonic sort of s[0..P), P a power of two.
__device__ void warp_bitonic(int32_t* s, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int32_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Per owned node: gather the node ids of every adjacent element, sort, unique
// (pattern.cpp:66-83, on node ids instead of DOFs — the d-expansion is exact).
// FILL=false: counts[v] = #unique; FILL=true: writes the list at ncol+nptr[v].
// Nodes with more than kNodeCap candidates are deferred to k_node_pattern_big.
template <bool FILL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_node_pattern(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj,
                   const int32_t* __restrict__ conn_k, int npe, int64_t n_own,
                   int64_t* __restrict__ counts, const int64_t* __restrict__ nptr,
                   int32_t* __restrict__ ncol, int32_t* __restrict__ big_list,
                   unsigned* __restrict__ n_big, unsigned* __restrict__ max_big) {
    __shared__ int32_t sh[kWarpsPerBlock][kNodeCap];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    int32_t* s = sh[w];
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n_own;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b0 = adj_ptr[v];
        const int64_t nc = (adj_ptr[v + 1] - b0) * npe;
        if (nc > kNodeCap) {
            if (!FILL && lane == 0) {
                big_list[atomicAdd(n_big, 1u)] = static_cast<int32_t>(v);
                atomicMax(max_big, static_cast<unsigned>(nc));
            }
            continue;
        }
        int P = 1;
        while (P < nc) P <<= 1;
        for (int i = lane; i < P; i += 32)
            s[i] = i < nc ? candidate(adj, conn_k, b0, npe, i) : INT32_MAX;
        __syncwarp();
        warp_bitonic(s, P, lane);
        int64_t out = FILL ? nptr[v] : 0;
        int total = 0;
        for (int i0 = 0; i0 < P; i0 += 32) {
            const int i = i0 + lane;
            const bool uniq = i < P && s[i] != INT32_MAX && (i == 0 || s[i] != s[i - 1]);
            const unsigned bal = __ballot_sync(0xffffffffu, uniq);
            if (FILL && uniq) ncol[out + total + __popc(bal & ((1u << lane) - 1u))] = s[i];
            total += __popc(bal);
        }
        if (!FILL && lane == 0) counts[v] = total;
        __syncwarp();
    }
}

// One pass instead of three (count, fill, slot map) for the common case - no high-valence node,
// rows of <= 256 column nodes (byte positions): the sorted unique list of a node is written to a
// scratch array at the node's candidate offset adj_ptr[v] * npe (an upper bound of its length,
// disjoint between nodes), its length to counts[v], and the node's slot-map rows posA straight
// from the list in shared memory (positions are row-relative, so they need no row pointer).
// After the row-pointer scan k_compact_lists copies the lists to ncol + nptr[v]. The caller
// falls back to the separate passes when a node was deferred or a row is longer than 256.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_node_pattern_fused(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj,
                         const int32_t* __restrict__ conn_k, int npe, int64_t n_own, int64_t* __restrict__ counts,
                         int32_t* __restrict__ scratch, int pstride, uint8_t* __restrict__ posA,
                         int32_t* __restrict__ big_list, unsigned* __restrict__ n_big,
                         unsigned* __restrict__ max_big) {
    __shared__ int32_t sh[kWarpsPerBlock][kNodeCap];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    int32_t* s = sh[w];
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n_own;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b0 = adj_ptr[v];
        const int64_t nc = (adj_ptr[v + 1] - b0) * npe;
        if (nc > kNodeCap) {
            if (lane == 0) {
                big_list[atomicAdd(n_big, 1u)] = static_cast<int32_t>(v);
                atomicMax(max_big, static_cast<unsigned>(nc));
            }
            continue;
        }
        int P = 1;
        while (P < nc) P <<= 1;
        for (int i = lane; i < P; i += 32)
            s[i] = i < nc ? candidate(adj, conn_k, b0, npe, i) : INT32_MAX;
        __syncwarp();
        warp_bitonic(s, P, lane);
        int total = 0;  // distinct values compacted to the front of s (a slot is never written
                        // before the step that reads it: total + rank <= i)
        for (int i0 = 0; i0 < P; i0 += 32) {
            const int i = i0 + lane;
            const int32_t x = i < P ? s[i] : INT32_MAX;  // (P may be smaller than a warp)
            const bool uniq = x != INT32_MAX && (i == 0 || x != s[i - 1]);
            const unsigned bal = __ballot_sync(0xffffffffu, uniq);
            __syncwarp();
            if (uniq) s[total + __popc(bal & ((1u << lane) - 1u))] = x;
            total += __popc(bal);
            __syncwarp();
        }
        if (lane == 0) counts[v] = total;
        int32_t* out = scratch + b0 * npe;
        for (int i = lane; i < total; i += 32) out[i] = s[i];
        if (total <= 256)
            for (int i = lane; i < nc; i += 32) {
                const int32_t u = candidate(adj, conn_k, b0, npe, i);
                int lo = 0, hi = total;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (s[mid] < u) lo = mid + 1;
                    else hi = mid;
                }
                const int k = i / npe;
                posA[(b0 + k) * pstride + (i - k * npe)] = static_cast<uint8_t>(lo);
            }
        __syncwarp();
    }
}

__global__ void k_compact_lists(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ scratch, int npe,
                                int64_t n_own, const int64_t* __restrict__ nptr, int32_t* __restrict__ ncol) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n_own;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t c0 = nptr[v];
        const int cnt = static_cast<int>(nptr[v + 1] - c0);
        const int32_t* src = scratch + adj_ptr[v] * npe;
        for (int i = lane; i < cnt; i += 32) ncol[c0 + i] = src[i];
    }
}

// Block-per-node fallback for high-valence nodes (dynamic shared memory).
template <bool FILL>
__global__ void k_node_pattern_big(const int64_t* __restrict__ adj_ptr,
                                   const int32_t* __restrict__ adj,
                                   const int32_t* __restrict__ conn_k, int npe,
                                   const int32_t* __restrict__ big_list, int64_t* __restrict__ counts,
                                   const int64_t* __restrict__ nptr, int32_t* __restrict__ ncol) {
    extern __shared__ int32_t s[];
    const int64_t v = big_list[blockIdx.x];
    const int64_t b0 = adj_ptr[v];
    const int64_t nc = (adj_ptr[v + 1] - b0) * npe;
    int P = 1;
    while (P < nc) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        s[i] = i < nc ? candidate(adj, conn_k, b0, npe, i) : INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int32_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0) {
        int64_t total = 0;
        const int64_t out = FILL ? nptr[v] : 0;
        for (int i = 0; i < P && s[i] != INT32_MAX; ++i)
            if (i == 0 || s[i] != s[i - 1]) {
                if (FILL) ncol[out + total] = s[i];
                ++total;
            }
        if (!FILL) counts[v] = total;
    }
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* __restrict__ a, int64_t n,
                                                   int32_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Slot map in adjacency order: for incidence k = (element, a) of node v and
// every node b of the element, the position of node b in v's sorted list.
// This is the per-entry locate() of scatter_element (assembly.hpp:84),
// resolved once for all entries sharing a (row node, column node) block.
template <class PosT>
__global__ void k_pos_adj(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj,
                          const int32_t* __restrict__ conn_k, int npe, int64_t n_own,
                          const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol,
                          int pstride, PosT* __restrict__ posA) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n_own;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b0 = adj_ptr[v];
        const int64_t nc = (adj_ptr[v + 1] - b0) * npe;
        const int32_t* list = ncol + nptr[v];
        const int64_t cnt = nptr[v + 1] - nptr[v];
        for (int64_t i = lane; i < nc; i += 32) {
            const int32_t u = candidate(adj, conn_k, b0, npe, i);
            const int64_t k = i / npe;
            posA[(b0 + k) * pstride + (i - k * npe)] = static_cast<PosT>(lower_bound_i32(list, cnt, u));
        }
    }
}

// Node-level CRAC run count (pattern.cpp:110-120 / formats.cpp:29 restated per
// node: column blocks of consecutive nodes merge into one run).
__global__ void k_node_runs(const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol,
                            int64_t n_own, int64_t* __restrict__ runs) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_own;
         v += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = 0;
        for (int64_t i = nptr[v]; i < nptr[v + 1]; ++i)
            if (i == nptr[v] || ncol[i] != ncol[i - 1] + 1) ++r;
        runs[v] = r;
    }
}

__global__ void k_max_i64(const int64_t* __restrict__ x, int64_t n, unsigned long long* out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, static_cast<unsigned long long>(x[i]));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_diff(const int64_t* __restrict__ ptr, int64_t n, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = ptr[i + 1] - ptr[i];
}

// CSR expansion of the node-level pattern (the SparsityPattern of
// pattern.hpp:29-35 for the owned block).
__global__ void k_expand_csr(const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol,
                             int64_t n_own, int d, int64_t node_begin, int64_t* __restrict__ row_ptr,
                             int64_t* __restrict__ cols) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n_own;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t cnt = nptr[v + 1] - nptr[v];
        const int64_t base = (int64_t)d * d * nptr[v];
        const int64_t rowlen = d * cnt;
        if (lane < d) row_ptr[v * d + lane] = base + lane * rowlen;
        if (v == n_own - 1 && lane == 0) row_ptr[n_own * d] = (int64_t)d * d * nptr[n_own];
        if (cols == nullptr) continue;  // row pointers only
        const int32_t* list = ncol + nptr[v];
        for (int64_t i = lane; i < d * rowlen; i += 32) {
            const int64_t k = i / rowlen;
            const int64_t q = i - k * rowlen;
            const int64_t p = q / d;
            cols[base + i] = (int64_t)list[p] * d + (q - p * d);
        }
    }
    (void)node_begin;
}

// CRAC arrays of the owned block (build_crac_arrays, formats.cpp:21-41):
// row_ptr in col_align entry units; (column start, values position) per run;
// the final (0, nnz) pair.
__global__ void k_expand_crac(const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol,
                              const int64_t* __restrict__ nrun_ptr, int64_t n_own, int d,
                              int64_t* __restrict__ crac_ptr, int64_t* __restrict__ col_align) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_own;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cnt = nptr[v + 1] - nptr[v];
        const int64_t nr = nrun_ptr[v + 1] - nrun_ptr[v];
        const int32_t* list = ncol + nptr[v];
        for (int k = 0; k < d; ++k) {
            const int64_t r = v * d + k;
            int64_t w = 2 * ((int64_t)d * nrun_ptr[v] + k * nr);
            crac_ptr[r] = w;
            const int64_t row_start = (int64_t)d * d * nptr[v] + (int64_t)k * d * cnt;
            for (int64_t p = 0; p < cnt; ++p)
                if (p == 0 || list[p] != list[p - 1] + 1) {
                    col_align[w++] = (int64_t)list[p] * d;
                    col_align[w++] = row_start + p * d;
                }
        }
        if (v == n_own - 1) {
            const int64_t tot = 2 * (int64_t)d * nrun_ptr[n_own];
            crac_ptr[n_own * d] = tot;
            col_align[tot] = 0;
            col_align[tot + 1] = (int64_t)d * d * nptr[n_own];
        }
    }
}

// External patterns: locate every element entry in the caller's CSR pattern
// (lower-bound search; the reference switches linear/binary at 30 entries,
// formats.hpp:196-199 — the found position is identical) or CRAC pattern
// (Listing 1 linear block search, formats.hpp:276-290). Each warp takes one
// incidence row at a time, its lanes the element's columns. Missing entries
// record the lowest (element, local row, local col) — the first one
// scatter_element would hit (assembly.hpp:80-88).
template <class PosT, bool CRAC>
__global__ void k_pos_external(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj,
                               const int32_t* __restrict__ conn_k, int npe, int64_t n_rows,
                               const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ cols,
                               const int64_t* __restrict__ crac_ptr,
                               const int64_t* __restrict__ col_align, int pstride,
                               PosT* __restrict__ posA, unsigned long long* __restrict__ miss) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n_rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b0 = adj_ptr[r];
        const int64_t nc = (adj_ptr[r + 1] - b0) * npe;
        const int64_t lo0 = row_ptr[r], hi0 = row_ptr[r + 1];
        for (int64_t i = lane; i < nc; i += 32) {
            const int64_t c = candidate(adj, conn_k, b0, npe, i);
            int64_t pos = -1;
            if (!CRAC) {
                int64_t lo = lo0, hi = hi0;
                while (lo < hi) {
                    const int64_t mid = lo + (hi - lo) / 2;
                    if (cols[mid] < c) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < hi0 && cols[lo] == c) pos = lo;
            } else {
                int64_t j = crac_ptr[r];
                const int64_t row_end = crac_ptr[r + 1];
                if (j != row_end) {
                    while (j + 2 < row_end && col_align[j + 2] <= c) j += 2;
                    const int64_t cs = col_align[j], vs = col_align[j + 1], ve = col_align[j + 3];
                    if (c >= cs && c < cs + (ve - vs)) pos = vs + (c - cs);
                }
            }
            if (pos < 0) {
                const int32_t entry = adj[b0 + i / npe];
                const int64_t e = entry / npe;  // external plans: K row == element id
                const int a = entry % npe;
                const int b = static_cast<int>(i % npe);
                atomicMin(miss, static_cast<unsigned long long>((e * npe + a) * npe + b));
                pos = lo0;
            }
            posA[(b0 + i / npe) * pstride + i % npe] = static_cast<PosT>(pos - lo0);
        }
    }
}

// ---- external patterns: validation and CRAC -> CSR view on the device --------------------
// (the reference trusts its own SparsityPattern; a caller's arrays are checked before any
// indexing. Codes are ordered like the checks: the lowest failing one is reported.)
enum ExtErr : unsigned {
    kExtPtr0 = 1, kExtPtrMono, kExtCracEven, kExtCracPos, kExtCracPast, kExtCracEmpty, kExtColRange,
    kExtColAsc, kExtOk = 0xffffffffu
};

const char* ext_err_text(unsigned c) {
    switch (c) {
        case kExtPtr0: return "row_ptr[0] must be 0";
        case kExtPtrMono: return "row_ptr not monotone";
        case kExtCracEven: return "CRAC row_ptr entries must be even";
        case kExtCracPos: return "CRAC runs: value positions must start at 0 and increase";
        case kExtCracPast: return "CRAC run extends past the last column";
        case kExtCracEmpty: return "CRAC pattern without runs must have nnz 0";
        case kExtColRange: return "pattern column outside the matrix";
        case kExtColAsc: return "pattern columns not strictly ascending within a row";
        default: return "malformed pattern";
    }
}

__global__ void k_ext_check_ptr(const int64_t* __restrict__ ptr, int64_t n_rows, bool crac,
                                unsigned* __restrict__ err) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = ptr[r];
        if (r == 0 && v != 0) atomicMin(err, (unsigned)kExtPtr0);
        if (r < n_rows && v > ptr[r + 1]) atomicMin(err, (unsigned)kExtPtrMono);
        if (crac && (v & 1)) atomicMin(err, (unsigned)kExtCracEven);
    }
}

// build_crac_arrays layout (formats.cpp:21-41): pairs (column start, values position), closed by
// (0, nnz). Every run's values position is the running count of the runs before it, so run
// lengths (next position - this one) must be positive and the first position 0.
__global__ void k_ext_check_runs(const int64_t* __restrict__ align, int64_t n_align, int64_t n_rows,
                                 unsigned* __restrict__ err) {
    const int64_t n_pairs = (n_align - 2) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_pairs;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cs = align[2 * j], vs = align[2 * j + 1], ve = align[2 * j + 3];
        if (cs < 0 || ve <= vs || (j == 0 && vs != 0)) atomicMin(err, (unsigned)kExtCracPos);
        else if (cs + (ve - vs) > n_rows) atomicMin(err, (unsigned)kExtCracPast);
    }
    if (n_pairs == 0 && blockIdx.x == 0 && threadIdx.x == 0 && align[1] != 0)
        atomicMin(err, (unsigned)kExtCracEmpty);
}

// CSR view of a (validated) CRAC pattern, for_each_in_row (formats.hpp:315-324): row r starts at
// the values position of its first run (an empty row: of the next run).
__global__ void k_ext_crac_csr_ptr(const int64_t* __restrict__ crac_ptr, const int64_t* __restrict__ align,
                                   int64_t n_rows, int64_t* __restrict__ csr_ptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_rows;
         r += (int64_t)gridDim.x * blockDim.x)
        csr_ptr[r] = align[crac_ptr[r] + 1];
}

__global__ void k_ext_crac_cols(const int64_t* __restrict__ align, int64_t n_pairs, int64_t* __restrict__ cols) {
    const int lane = threadIdx.x & 31;  // a warp per run
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n_pairs;
         j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t cs = align[2 * j], vs = align[2 * j + 1], len = align[2 * j + 3] - vs;
        for (int64_t k = lane; k < len; k += 32) cols[vs + k] = cs + k;
    }
}

// Rows of the CSR view: columns inside the matrix and strictly ascending (a warp per row);
// also the int32 column copy the plan keeps and the longest row.
__global__ void k_ext_check_rows(const int64_t* __restrict__ ptr, const int64_t* __restrict__ cols,
                                 int64_t n_rows, int32_t* __restrict__ ncol, unsigned* __restrict__ err,
                                 unsigned long long* __restrict__ max_len) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n_rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t lo = ptr[r], hi = ptr[r + 1];
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const int64_t c = cols[i];
            if (c < 0 || c >= n_rows) atomicMin(err, (unsigned)kExtColRange);
            else if (i > lo && cols[i - 1] >= c) atomicMin(err, (unsigned)kExtColAsc);
            ncol[i] = static_cast<int32_t>(c);
        }
        if (lane == 0) atomicMax(max_len, static_cast<unsigned long long>(hi - lo));
    }
}

// Colour-ordered incidences (FEA_DET_COLOUR as a segmented reduction): keys for a
// two-pass LSD stable sort, first by colour, then by node — each node's incidences end up
// in ascending (colour, element id).
__global__ void k_node_of(const int64_t* __restrict__ adj_ptr, int64_t n_own, int32_t* __restrict__ node_of) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_own;
         v += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = adj_ptr[v]; k < adj_ptr[v + 1]; ++k) node_of[k] = static_cast<int32_t>(v);
}

// colour of every K row from the colour of every kept element (rows of other elements: 0)
__global__ void k_colour_of_krow(const int32_t* __restrict__ elem_krow, const int32_t* __restrict__ col, int64_t E,
                                 int32_t* __restrict__ colour_of_krow) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        colour_of_krow[elem_krow[e]] = col[e];
}

// find_colour_conflict (colouring.cpp:91-119) as a yes / no question: does any owned node have two
// different incident elements of one colour? (The offending pair is then named by the host scan,
// in the reference's order; a valid colouring - the usual case - never reaches it.)
__global__ void k_colour_conflict(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj, int64_t n_own,
                                  int npe, const int32_t* __restrict__ colour_of_krow, unsigned* __restrict__ flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_own; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b0 = adj_ptr[v];
        const int n = static_cast<int>(adj_ptr[v + 1] - b0);
        bool bad = false;
        for (int i = 1; i < n && !bad; ++i) {
            const int32_t ki = adj[b0 + i] / npe;
            const int32_t ci = colour_of_krow[ki];
            for (int j = 0; j < i; ++j) {
                const int32_t kj = adj[b0 + j] / npe;
                if (kj != ki && colour_of_krow[kj] == ci) {
                    bad = true;
                    break;
                }
            }
        }
        if (bad) atomicOr(flag, 1u);
    }
}

__global__ void k_colour_keys(const int32_t* __restrict__ adj, int64_t n_adj, int npe,
                              const int32_t* __restrict__ colour_of_krow, uint32_t* __restrict__ keys,
                              int32_t* __restrict__ vals) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_adj;
         k += (int64_t)gridDim.x * blockDim.x) {
        keys[k] = static_cast<uint32_t>(colour_of_krow[adj[k] / npe]);
        vals[k] = static_cast<int32_t>(k);
    }
}

__global__ void k_gather_keys(const int32_t* __restrict__ node_of, const int32_t* __restrict__ perm,
                              int64_t n, uint32_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = static_cast<uint32_t>(node_of[perm[i]]);
}

__global__ void k_permute_incidences(const int32_t* __restrict__ perm, int64_t n, int row_bytes,
                                     const int32_t* __restrict__ adj, const unsigned char* __restrict__ posA,
                                     int32_t* __restrict__ adjC, unsigned char* __restrict__ posAC) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = perm[i];
        adjC[i] = adj[k];
        const uint32_t* src = reinterpret_cast<const uint32_t*>(posA + k * row_bytes);
        uint32_t* dst = reinterpret_cast<uint32_t*>(posAC + i * row_bytes);
        for (int w = 0; w < row_bytes / 4; ++w) dst[w] = src[w];
    }
}

// Locality of the node-id traversal for the gather: does node v share an element with
// node v+1? (two-pointer merge of the ascending incidence lists). keys = lowest element.
__global__ void k_node_share(const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj,
                             int npe, int64_t n_own, unsigned long long* shared,
                             uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_own;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a0 = adj_ptr[v], a1 = adj_ptr[v + 1];
        keys[v] = a1 > a0 ? static_cast<uint32_t>(adj[a0] / npe) : 0xffffffffu;
        vals[v] = static_cast<int32_t>(v);
        if (v + 1 < n_own) {
            int64_t i = a0, j = a1;
            const int64_t j1 = adj_ptr[v + 2];
            bool sh = false;
            while (i < a1 && j < j1 && !sh) {
                const int32_t ei = adj[i] / npe, ej = adj[j] / npe;
                if (ei == ej) sh = true;
                else if (ei < ej) ++i;
                else ++j;
            }
            if (sh) atomicAdd(shared, 1ull);
        }
    }
}

// Jones-Plassmann colouring (GPU colouring): every round, each
// uncoloured element whose seeded priority beats all uncoloured elements sharing an (owned)
// node takes the smallest colour no coloured neighbour uses. Two neighbours are never local
// maxima in the same round, so colours read from neighbours are stable within a round.
__global__ void k_jp_prio(const int64_t* __restrict__ elem_id, int64_t E, uint64_t seed,
                          uint64_t* __restrict__ prio, int32_t* __restrict__ colour) {
    for (int64_t le = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; le < E;
         le += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + static_cast<uint64_t>(elem_id[le]) + 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        prio[le] = (z & ~0xffffffffULL) | static_cast<uint32_t>(le);  // ties broken by index
        colour[le] = -1;
    }
}

__global__ void k_jp_round(const int32_t* __restrict__ conn_k, const int32_t* __restrict__ elem_krow,
                           const int32_t* __restrict__ k2l, int64_t E, int npe, int64_t node_begin,
                           int64_t node_end, const int64_t* __restrict__ adj_ptr,
                           const int32_t* __restrict__ adj, const uint64_t* __restrict__ prio,
                           int32_t* __restrict__ colour, unsigned long long* __restrict__ remaining) {
    for (int64_t le = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; le < E;
         le += (int64_t)gridDim.x * blockDim.x) {
        if (colour[le] >= 0) continue;
        const uint64_t mine = prio[le];
        const int32_t* c = conn_k + static_cast<int64_t>(elem_krow[le]) * npe;
        uint64_t used[2] = {0, 0};
        bool local_max = true;
        for (int a = 0; a < npe && local_max; ++a) {
            const int64_t v = c[a];
            if (v < node_begin || v >= node_end) continue;
            const int64_t lv = v - node_begin;
            for (int64_t k = adj_ptr[lv]; k < adj_ptr[lv + 1]; ++k) {
                const int32_t kr = adj[k] / npe;
                const int64_t o = k2l ? k2l[kr] : kr;
                if (o == le) continue;
                const int32_t oc = colour[o];
                if (oc < 0) {
                    if (prio[o] > mine) { local_max = false; break; }
                } else if (oc < 128) {
                    used[oc >> 6] |= 1ull << (oc & 63);
                }
            }
        }
        if (!local_max) {
            atomicAdd(remaining, 1ull);
            continue;
        }
        const int c0 = __ffsll(static_cast<long long>(~used[0]));
        colour[le] = c0 ? c0 - 1 : 64 + __ffsll(static_cast<long long>(~used[1])) - 1;
    }
}

// ---------------------------------------------------------------------------
// Host orchestration
// ---------------------------------------------------------------------------

struct Tmp {
    DevBuf buf;
    template <class T>
    T* alloc(size_t n) {
        buf.alloc(n * sizeof(T));
        return buf.as<T>();
    }
};

// Host -> device copy of a large caller array. The reference interface hands over int64 DOFs
// in ordinary (pageable) memory - 3.2 GB on config 5 - which a plain cudaMemcpy moves through
// the driver's single staging thread at 5-9 GB/s (360-700 ms, five times the whole symbolic
// phase on the device). Here a few host threads copy interleaved 8 MiB chunks into their own
// pinned double buffers and issue the bulk transfers on their own streams, so the host-side
// memcpy runs in parallel and overlaps the PCIe transfer. Pinned sources and small arrays take
// the plain copy. The copy has completed when the function returns.
void upload_host(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t kChunk = size_t{8} << 20;
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const unsigned hw = std::thread::hardware_concurrency();
    const int T = static_cast<int>(std::min<size_t>({size_t{8}, hw > 1 ? hw / 2 : 1, bytes / (4 * kChunk)}));
    if (pinned || T < 2 || std::getenv("FEA_PLAIN_UPLOAD")) {
        FEA_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        FEA_CK(cudaStreamSynchronize(s));
        return;
    }
    int dev = 0;
    FEA_CK(cudaGetDevice(&dev));
    const size_t n_chunks = (bytes + kChunk - 1) / kChunk;
    std::vector<cudaError_t> err(static_cast<size_t>(T), cudaSuccess);
    auto worker = [&](int t) {
        cudaError_t& e = err[static_cast<size_t>(t)];
        auto ok = [&](cudaError_t r) {
            if (e == cudaSuccess && r != cudaSuccess) e = r;
            return e == cudaSuccess;
        };
        unsigned char* stage[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        cudaStream_t st = nullptr;
        if (ok(cudaSetDevice(dev)) && ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking))) {
            for (int b = 0; b < 2; ++b) {
                ok(cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), kChunk, cudaHostAllocDefault));
                ok(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
            }
            int b = 0;
            for (size_t c = static_cast<size_t>(t); c < n_chunks && e == cudaSuccess; c += static_cast<size_t>(T), b ^= 1) {
                const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
                if (!ok(cudaEventSynchronize(ev[b]))) break;  // the buffer's previous transfer
                std::memcpy(stage[b], static_cast<const unsigned char*>(src) + off, len);
                ok(cudaMemcpyAsync(static_cast<unsigned char*>(dst) + off, stage[b], len, cudaMemcpyHostToDevice, st));
                ok(cudaEventRecord(ev[b], st));
            }
            ok(cudaStreamSynchronize(st));
        }
        for (int b = 0; b < 2; ++b) {
            if (ev[b]) cudaEventDestroy(ev[b]);
            if (stage[b]) cudaFreeHost(stage[b]);
        }
        if (st) cudaStreamDestroy(st);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (std::thread& th : pool) th.join();
    for (cudaError_t e : err) FEA_CK(e);
}

// Upload (or alias) the element DOF array.
const int64_t* device_dofs(const int64_t* elem_dofs, int64_t n, DevBuf& hold, cudaStream_t s) {
    if (n == 0) return nullptr;
    if (is_device_ptr(elem_dofs)) return elem_dofs;
    hold.alloc(n * sizeof(int64_t));
    upload_host(hold.p, elem_dofs, n * sizeof(int64_t), s);
    return hold.as<int64_t>();
}

// Node->element incidences + adjacency (shared by own and external patterns).
void build_adjacency(fea_plan* p, cudaStream_t s) {
    const int64_t items = p->E * p->npe;
    FEA_REQUIRE(items < (int64_t{1} << 31) && p->krows() * p->npe < (int64_t{1} << 31),
                FEA_ERR_INVALID, "more than 2^31 element-node incidences are not supported");
    DevBuf counts_b;
    counts_b.alloc((p->n_own + 1) * sizeof(int64_t));
    FEA_CK(cudaMemsetAsync(counts_b.p, 0, counts_b.bytes, s));
    DevBuf keys_in, vals_in, keys_out, vals_out;
    keys_in.alloc(items * 4);
    vals_in.alloc(items * 4);
    keys_out.alloc(items * 4);
    vals_out.alloc(items * 4);
    if (items > 0) {
        k_emit_incidences<<<grid_for(items, 256), 256, 0, s>>>(
            p->conn_k.as<int32_t>(), p->elem_krow.as<int32_t>(), p->E, p->npe, p->node_begin,
            p->node_end, keys_in.as<uint32_t>(), vals_in.as<int32_t>(),
            counts_b.as<unsigned long long>());
        FEA_CK(cudaGetLastError());
        const int end_bit = bits_for(static_cast<uint64_t>(p->n_own));
        radix_sort_pairs(keys_in.as<uint32_t>(), keys_out.as<uint32_t>(), vals_in.as<int32_t>(),
                         vals_out.as<int32_t>(), items, 0, end_bit, s);
    }
    p->adj_ptr.alloc((p->n_own + 1) * sizeof(int64_t));
    exclusive_sum(counts_b.as<int64_t>(), p->adj_ptr.as<int64_t>(), p->n_own + 1, s);
    FEA_CK(cudaMemcpyAsync(&p->n_adj, p->adj_ptr.as<int64_t>() + p->n_own, sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    p->adj.alloc(p->n_adj * 4 + 64);  // slack: 16B-rounded bulk copies of adjacency slices
    if (p->n_adj > 0)
        FEA_CK(cudaMemcpyAsync(p->adj.p, vals_out.p, p->n_adj * 4, cudaMemcpyDeviceToDevice, s));
    // largest node incidence count (reporting / sizing)
    {
        DevBuf cnt, mx;
        cnt.alloc(p->n_own * 8 + 8);
        mx.alloc(8);
        FEA_CK(cudaMemsetAsync(mx.p, 0, 8, s));
        if (p->n_own > 0) {
            k_diff<<<grid_for(p->n_own, 256), 256, 0, s>>>(p->adj_ptr.as<int64_t>(), p->n_own,
                                                           cnt.as<int64_t>());
            k_max_i64<<<grid_for(p->n_own, 256), 256, 0, s>>>(cnt.as<int64_t>(), p->n_own,
                                                              mx.as<unsigned long long>());
            FEA_CK(cudaGetLastError());
        }
        unsigned long long h = 0;
        FEA_CK(cudaMemcpyAsync(&h, mx.p, 8, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        p->max_adj = static_cast<int64_t>(h);
    }
}

void finish_counts(fea_plan* p, DevBuf& counts, cudaStream_t s) {
    p->nptr.alloc((p->n_own + 1) * sizeof(int64_t));
    exclusive_sum(counts.as<int64_t>(), p->nptr.as<int64_t>(), p->n_own + 1, s);
    DevBuf mx;
    mx.alloc(8);
    FEA_CK(cudaMemsetAsync(mx.p, 0, 8, s));
    if (p->n_own > 0)
        k_max_i64<<<grid_for(p->n_own, 256), 256, 0, s>>>(counts.as<int64_t>(), p->n_own,
                                                          mx.as<unsigned long long>());
    FEA_CK(cudaGetLastError());
    unsigned long long h = 0;
    FEA_CK(cudaMemcpyAsync(&h, mx.p, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(&p->nnz_nodes, p->nptr.as<int64_t>() + p->n_own, 8,
                           cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    FEA_REQUIRE(h <= 65536, FEA_ERR_INVALID,
                "a pattern row has more than 65536 column nodes (position map limit)");
    p->max_cnt = static_cast<int32_t>(h);
    p->pos_bytes = h <= 256 ? 1 : 2;
    p->pstride = ((p->npe * p->pos_bytes + 3) / 4 * 4) / p->pos_bytes;
    p->nnz = static_cast<int64_t>(p->d) * p->d * p->nnz_nodes;
}

// Gather traversal order. Node-id order when consecutive nodes already share elements
// (structured numbering); otherwise (permuted node ids) nodes sorted by their lowest
// incident element, so the row blocks an element contributes to its nodes are read close
// together in time and its 128 B lines are served from L2 (measured on cfg3: 4.2x DRAM
// read amplification without it). Only for row blocks smaller than a line (d*m*8 < 128).
void build_node_order(fea_plan* p, cudaStream_t s) {
    p->node_order.reset();
    if (p->n_own < 2 || p->d * p->m * 8 >= 128 || std::getenv("FEA_NODE_ORDER_ID")) return;
    DevBuf keys, vals, keys2, cnt;
    keys.alloc(p->n_own * 4);
    vals.alloc(p->n_own * 4);
    keys2.alloc(p->n_own * 4);
    cnt.alloc(8);
    FEA_CK(cudaMemsetAsync(cnt.p, 0, 8, s));
    k_node_share<<<grid_for(p->n_own, 256), 256, 0, s>>>(p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(),
                                                         p->npe, p->n_own, cnt.as<unsigned long long>(),
                                                         keys.as<uint32_t>(), vals.as<int32_t>());
    FEA_CK(cudaGetLastError());
    unsigned long long shared = 0;
    FEA_CK(cudaMemcpyAsync(&shared, cnt.p, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    if (2 * static_cast<int64_t>(shared) >= p->n_own - 1) return;
    p->node_order.alloc(p->n_own * 4);
    radix_sort_pairs(keys.as<uint32_t>(), keys2.as<uint32_t>(), vals.as<int32_t>(),
                     p->node_order.as<int32_t>(), p->n_own, 0, 32, s);
    FEA_CK(cudaStreamSynchronize(s));
}

__global__ void k_trav_count(const int32_t* __restrict__ order, const int64_t* __restrict__ adj_ptr,
                             const int64_t* __restrict__ nptr, int64_t n_own, int64_t* __restrict__ cnt,
                             int64_t* __restrict__ meta) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_own;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = order != nullptr ? order[t] : t;
        cnt[t] = adj_ptr[v + 1] - adj_ptr[v];
        meta[t] = (nptr[v] << 20) | (nptr[v + 1] - nptr[v]);
    }
}

__global__ void k_trav_records(const int32_t* __restrict__ order, const int64_t* __restrict__ adj_ptr,
                               const int32_t* __restrict__ adj, const uint32_t* __restrict__ pos_words,
                               int pw, int rw, const int64_t* __restrict__ tptr, int64_t n_own,
                               int32_t* __restrict__ rec) {
    // one warp per traversal position: lanes copy the node's records
    const int lane = threadIdx.x & 31;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_own;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t v = order != nullptr ? order[t] : t;
        const int64_t a0 = adj_ptr[v], n = adj_ptr[v + 1] - a0, r0 = tptr[t];
        for (int64_t k = lane; k < n; k += 32) {
            int32_t* r = rec + (r0 + k) * rw;
            r[0] = adj[a0 + k];
            for (int w = 0; w < pw; ++w) r[1 + w] = static_cast<int32_t>(pos_words[(a0 + k) * pw + w]);
            for (int w = pw + 1; w < rw; ++w) r[w] = 0;
        }
    }
}

void build_lane_slots(fea_plan* p, cudaStream_t s);

// d = 1 sorted gather with a traversal order: incidence records in traversal order
void build_traversal(fea_plan* p, cudaStream_t s) {
    p->trav_ptr.reset();
    p->trav_meta.reset();
    p->trav_rec.reset();
    // (also without a traversal order: the records then follow node id order and the d = 1
    // kernels still save the adj_ptr -> adj / posA round trip per node, cfg1)
    if (p->d != 1 || p->npe > 32 || p->d1_disabled || std::getenv("FEA_NO_TRAVERSAL_RECORDS")) return;
    const int pw = p->pstride * p->pos_bytes / 4;
    const int rw = pw == 1 ? 2 : (pw + 4) & ~3;
    DevBuf cnt;
    cnt.alloc((p->n_own + 1) * 8);
    FEA_CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes, s));
    p->trav_meta.alloc(p->n_own * 8);
    k_trav_count<<<grid_for(p->n_own, 256), 256, 0, s>>>(p->node_order.as<int32_t>(), p->adj_ptr.as<int64_t>(),
                                                         p->nptr.as<int64_t>(), p->n_own, cnt.as<int64_t>(),
                                                         p->trav_meta.as<int64_t>());
    FEA_CK(cudaGetLastError());
    p->trav_ptr.alloc((p->n_own + 1) * 8);
    exclusive_sum(cnt.as<int64_t>(), p->trav_ptr.as<int64_t>(), p->n_own + 1, s);
    p->trav_rec.alloc(std::max<int64_t>(p->n_adj, 1) * rw * 4);
    k_trav_records<<<grid_for(p->n_own * 32, 256), 256, 0, s>>>(
        p->node_order.as<int32_t>(), p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(),
        static_cast<const uint32_t*>(p->posA.p), pw, rw, p->trav_ptr.as<int64_t>(), p->n_own,
        p->trav_rec.as<int32_t>());
    FEA_CK(cudaGetLastError());
    p->trav_rw = rw;
    build_lane_slots(p, s);
    FEA_CK(cudaStreamSynchronize(s));
}

// --- lane-owned slots (k_gather_d1s: d = 1, npe = 4, rows of <= 16 nodes) ---------------------
// One thread per traversal position gives every slot of its node's row to one of the 4 lanes of
// the node's group so that the 4 columns of every incident element fall on 4 distinct lanes.
// The node's own (diagonal) slot shares an element with every other slot that any element
// touches, so it takes lane 0 alone; the rest is a 3-colouring of the node's link (DSATUR: on a
// Kuhn tet mesh the link is a triangulated sphere and every step after the first triangle is
// forced). The three classes are renamed by size (smallest = lane 1), slots of one lane take
// that lane's accumulators in slot order. A node that cannot be coloured, or needs more than 8
// accumulators on one lane, sets the plan's fail flag and the shared-memory fold stays in use.
// stats: [0] fail, [1..3] most accumulators on lane 1..3, [4] most on any lane,
// [5] largest entry - 4 * lowest K row of the node (width of the compact record's entry field)
__global__ void k_lane_colour(const int64_t* __restrict__ tptr, const int64_t* __restrict__ tmeta,
                              const int2* __restrict__ trec, int64_t n_own, uint8_t* __restrict__ slotmap,
                              int4* __restrict__ hdr, int* __restrict__ stats) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_own;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a0 = tptr[t];
        const int n = static_cast<int>(tptr[t + 1] - a0);
        const int64_t mt = tmeta[t];
        const int rl = static_cast<int>(mt & 0xfffff);
        if (rl > 16) {
            atomicOr(stats, 1);
            continue;
        }
        uint32_t adjm[16];
        uint8_t used[16], col[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) adjm[i] = 0, used[i] = 0, col[i] = 0xff;
        bool bad = false;
        int diag = -1;
        uint32_t emin = 0xffffffffu, emax = 0;
        for (int k = 0; k < n; ++k) {
            const int2 r = trec[a0 + k];
            const uint32_t w = static_cast<uint32_t>(r.y);
            uint32_t m = 0;
            for (int b = 0; b < 4; ++b) {
                const uint32_t sl = (w >> (8 * b)) & 0xffu;
                if (sl >= static_cast<uint32_t>(rl)) bad = true;
                m |= 1u << (sl & 15);
            }
            if (__popc(m) != 4) bad = true;
            for (int b = 0; b < 4; ++b) adjm[(w >> (8 * b)) & 15] |= m;
            const int dg = static_cast<int>((w >> (8 * (r.x & 3))) & 15u);  // the node's own column
            if (diag >= 0 && dg != diag) bad = true;
            diag = dg;
            emin = min(emin, static_cast<uint32_t>(r.x));
            emax = max(emax, static_cast<uint32_t>(r.x));
        }
        int cnt[4] = {0, 0, 0, 0};
        if (diag >= 0 && !bad) {
            col[diag] = 0;
            cnt[0] = 1;
            uint32_t nb = adjm[diag] & ~(1u << diag);
            while (nb) {
                const int u = __ffs(nb) - 1;
                nb &= nb - 1;
                used[u] |= 1;
            }
        }
        for (int it = cnt[0]; it < rl && !bad; ++it) {
            int best = -1, bkey = -1;
            for (int sl = 0; sl < rl; ++sl) {
                if (col[sl] != 0xff) continue;
                const int key = __popc(used[sl]) * 64 + __popc(adjm[sl]);
                if (key > bkey) bkey = key, best = sl;
            }
            int c = -1;
            for (int q = 1; q < 4; ++q)
                if (!((used[best] >> q) & 1) && (c < 0 || cnt[q] < cnt[c])) c = q;
            if (c < 0) {
                bad = true;
                break;
            }
            col[best] = static_cast<uint8_t>(c);
            ++cnt[c];
            uint32_t nb = adjm[best] & ~(1u << best);
            while (nb) {
                const int u = __ffs(nb) - 1;
                nb &= nb - 1;
                used[u] |= static_cast<uint8_t>(1u << c);
            }
        }
        if (bad || cnt[1] > 8 || cnt[2] > 8 || cnt[3] > 8) {
            atomicOr(stats, 1);
            continue;
        }
        // rename classes 1..3 by size (ties by class number): ren[old] = new lane
        int ren[4] = {0, 1, 2, 3};
        for (int i = 1; i < 4; ++i) {
            int rank = 1;
            for (int j = 1; j < 4; ++j)
                if (j != i && (cnt[j] < cnt[i] || (cnt[j] == cnt[i] && j < i))) ++rank;
            ren[i] = rank;
        }
        uint32_t lw[4] = {0, 0, 0, 0};
        int nq[4] = {0, 0, 0, 0};
        for (int sl = 0; sl < 16; ++sl) {
            uint8_t cq = 0;
            if (sl < rl) {
                const int c = ren[col[sl]], q = nq[c]++;
                lw[c] |= static_cast<uint32_t>(sl) << (4 * q);
                cq = static_cast<uint8_t>(c | (q << 2));
            }
            slotmap[t * 16 + sl] = cq;
        }
        atomicMax(stats + 1, nq[1]);
        atomicMax(stats + 2, nq[2]);
        atomicMax(stats + 3, nq[3]);
        atomicMax(stats + 4, max(max(nq[0], nq[1]), max(nq[2], nq[3])));
        const uint32_t base = n > 0 ? (emin & ~3u) : 0u;
        if (n > 0) atomicMax(stats + 5, static_cast<int>(min(emax - base, 0x7fffffffu)));
        const int64_t li = ((mt >> 20) << 20) | nq[0] | (nq[1] << 4) | (nq[2] << 8) | (nq[3] << 12) |
                           (static_cast<int64_t>(lw[0] & 15u) << 16);
        const int64_t an = a0 | (static_cast<int64_t>(n) << 40);
        hdr[2 * t] = make_int4(static_cast<int>(li & 0xffffffff), static_cast<int>(li >> 32),
                               static_cast<int>(an & 0xffffffff), static_cast<int>(an >> 32));
        hdr[2 * t + 1] = make_int4(static_cast<int>(base), static_cast<int>(lw[1]), static_cast<int>(lw[2]),
                                   static_cast<int>(lw[3]));
    }
}

// Records of the lane-owned gather from the traversal records {entry, position bytes}. Word
// layout (LSB first): for lanes 1, 2, 3 in turn the element column the lane loads (2 bits) and
// its accumulator (wq[c-1] bits, plan-wide widths), then - compact 4-byte form only - entry -
// 4 * the node's lowest K row. Lane 0 takes the node's own column (entry & 3) and accumulator
// 0. The 8-byte form keeps the entry in its own word.
struct LaneFmt {
    int wq[3];
    int sh_e;  // 6 + wq[0] + wq[1] + wq[2]: first bit of the entry offset
};
template <bool REC4>
__global__ void k_lane_records(const int64_t* __restrict__ tptr, const int2* __restrict__ trec,
                               const uint8_t* __restrict__ slotmap, const int4* __restrict__ hdr, int64_t n_own,
                               LaneFmt f, void* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_own;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a0 = tptr[t], n = tptr[t + 1] - a0;
        const uint32_t base = static_cast<uint32_t>(hdr[2 * t + 1].x);
        for (int64_t k = lane; k < n; k += 32) {
            const int2 r = trec[a0 + k];
            uint32_t word = 0;
            for (int b = 0; b < 4; ++b) {
                const uint32_t sl = (static_cast<uint32_t>(r.y) >> (8 * b)) & 15u;
                const uint32_t cq = slotmap[t * 16 + sl];
                const int c = static_cast<int>(cq & 3u);
                if (c == 0) continue;  // the node's own column: b = entry & 3, accumulator 0
                int off = 0;
                for (int j = 0; j < c - 1; ++j) off += 2 + f.wq[j];
                word |= (static_cast<uint32_t>(b) | ((cq >> 2) << 2)) << off;
            }
            if (REC4) {
                word |= (static_cast<uint32_t>(r.x) - base) << f.sh_e;
                static_cast<uint32_t*>(out)[a0 + k] = word;
            } else {
                static_cast<int2*>(out)[a0 + k] = make_int2(r.x, static_cast<int>(word));
            }
        }
    }
}

void build_lane_records(fea_plan* p, const DevBuf& trec, DevBuf& out, cudaStream_t s) {
    out.reset();
    if (!p->ln_ok || !trec.p) return;
    const LaneFmt f = {{p->ln_wq[0], p->ln_wq[1], p->ln_wq[2]}, 6 + p->ln_wq[0] + p->ln_wq[1] + p->ln_wq[2]};
    out.alloc(std::max<int64_t>(p->n_adj, 1) * (p->ln_rec4 ? 4 : 8));
    auto kern = p->ln_rec4 ? k_lane_records<true> : k_lane_records<false>;
    kern<<<grid_for(p->n_own * 32, 256), 256, 0, s>>>(p->trav_ptr.as<int64_t>(), reinterpret_cast<const int2*>(trec.p),
                                                      p->ln_slot.as<uint8_t>(), p->ln_hdr.as<int4>(), p->n_own, f,
                                                      out.p);
    FEA_CK(cudaGetLastError());
}

void build_lane_slots(fea_plan* p, cudaStream_t s) {
    p->ln_slot.reset();
    p->ln_hdr.reset();
    p->ln_rec.reset();
    p->ln_recC.reset();
    p->ln_ok = false;
    p->ln_rec4 = false;
    p->ln_q = 0;
    if (!p->trav_rec.p || p->d != 1 || p->npe != 4 || p->dup_nodes || p->pos_bytes != 1 || p->trav_rw != 2 ||
        p->max_cnt > 16 || p->max_adj >= 65536 || p->n_own == 0 || p->n_adj == 0 || p->kn.d1_no_lane)
        return;
    p->ln_slot.alloc(p->n_own * 16);
    p->ln_hdr.alloc(p->n_own * 32);
    DevBuf stats;
    stats.alloc(6 * 4);
    FEA_CK(cudaMemsetAsync(stats.p, 0, stats.bytes, s));
    k_lane_colour<<<grid_for(p->n_own, 128), 128, 0, s>>>(
        p->trav_ptr.as<int64_t>(), p->trav_meta.as<int64_t>(), reinterpret_cast<const int2*>(p->trav_rec.p),
        p->n_own, p->ln_slot.as<uint8_t>(), p->ln_hdr.as<int4>(), stats.as<int>());
    FEA_CK(cudaGetLastError());
    int h[6] = {0, 0, 0, 0, 0, 0};
    FEA_CK(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    if (h[0] != 0) {
        p->ln_slot.reset();
        p->ln_hdr.reset();
        return;
    }
    p->ln_ok = true;
    p->ln_q = std::max(h[4], 1);
    int bits = 6;
    for (int c = 0; c < 3; ++c) {
        p->ln_wq[c] = h[1 + c] <= 1 ? 0 : bits_for(static_cast<uint64_t>(h[1 + c] - 1));
        bits += p->ln_wq[c];
    }
    // compact records when the entry offset fits next to the lane fields
    p->ln_rec4 = !p->kn.d1_rec8 && static_cast<uint64_t>(h[5]) < (uint64_t{1} << (32 - bits));
    build_lane_records(p, p->trav_rec, p->ln_rec, s);
}

void build_runs(fea_plan* p, cudaStream_t s) {
    DevBuf runs;
    runs.alloc((p->n_own + 1) * sizeof(int64_t));
    FEA_CK(cudaMemsetAsync(runs.p, 0, runs.bytes, s));
    if (p->n_own > 0)
        k_node_runs<<<grid_for(p->n_own, 256), 256, 0, s>>>(p->nptr.as<int64_t>(),
                                                            p->ncol.as<int32_t>(), p->n_own,
                                                            runs.as<int64_t>());
    FEA_CK(cudaGetLastError());
    p->nrun_ptr.alloc((p->n_own + 1) * sizeof(int64_t));
    exclusive_sum(runs.as<int64_t>(), p->nrun_ptr.as<int64_t>(), p->n_own + 1, s);
    int64_t nr = 0;
    FEA_CK(cudaMemcpyAsync(&nr, p->nrun_ptr.as<int64_t>() + p->n_own, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    p->n_runs = nr * p->d;
}

void build_own_pattern(fea_plan* p, cudaStream_t s) {
    StageTrace tr;
    const unsigned blocks = grid_for(p->n_own * 32, kWarpsPerBlock * 32);
    DevBuf counts, big, nbig, maxbig, scratch;
    counts.alloc((p->n_own + 1) * sizeof(int64_t));
    FEA_CK(cudaMemsetAsync(counts.p, 0, counts.bytes, s));
    big.alloc((p->n_own + 1) * 4);
    nbig.alloc(4);
    maxbig.alloc(4);
    FEA_CK(cudaMemsetAsync(nbig.p, 0, 4, s));
    FEA_CK(cudaMemsetAsync(maxbig.p, 0, 4, s));
    // fused pass (k_node_pattern_fused): lists to scratch, byte positions to posA
    const bool try_fused = std::getenv("FEA_PLAN_NO_FUSED") == nullptr;
    const int pstride1 = (p->npe + 3) / 4 * 4;
    if (try_fused) {
        scratch.alloc(std::max<int64_t>(p->n_adj * p->npe, 1) * 4);
        p->posA.alloc(p->n_adj * pstride1 + 64);
        FEA_CK(cudaMemsetAsync(p->posA.p, 0, p->posA.bytes, s));
    }
    if (p->n_own > 0) {
        if (try_fused)
            k_node_pattern_fused<<<blocks, kWarpsPerBlock * 32, 0, s>>>(
                p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe, p->n_own,
                counts.as<int64_t>(), scratch.as<int32_t>(), pstride1, p->posA.as<uint8_t>(), big.as<int32_t>(),
                nbig.as<unsigned>(), maxbig.as<unsigned>());
        else
            k_node_pattern<false><<<blocks, kWarpsPerBlock * 32, 0, s>>>(
                p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe,
                p->n_own, counts.as<int64_t>(), nullptr, nullptr, big.as<int32_t>(),
                nbig.as<unsigned>(), maxbig.as<unsigned>());
    }
    FEA_CK(cudaGetLastError());
    unsigned h_nbig = 0, h_maxbig = 0;
    FEA_CK(cudaMemcpyAsync(&h_nbig, nbig.p, 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(&h_maxbig, maxbig.p, 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    size_t big_smem = 0;
    if (h_nbig > 0) {
        unsigned P = 1;
        while (P < h_maxbig) P <<= 1;
        big_smem = static_cast<size_t>(P) * 4;
        FEA_REQUIRE(big_smem <= 200 * 1024, FEA_ERR_INVALID,
                    "node valence too high for the symbolic phase (> 51200 candidate nodes)");
        FEA_CK(cudaFuncSetAttribute(k_node_pattern_big<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
        FEA_CK(cudaFuncSetAttribute(k_node_pattern_big<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
        k_node_pattern_big<false><<<h_nbig, 256, big_smem, s>>>(
            p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe,
            big.as<int32_t>(), counts.as<int64_t>(), nullptr, nullptr);
        FEA_CK(cudaGetLastError());
    }
    tr.mark(try_fused ? "node pattern (fused)" : "node pattern (count)", s);
    finish_counts(p, counts, s);
    tr.mark("row pointer scan", s);
    p->ncol.alloc(p->nnz_nodes * 4);
    const bool fused = try_fused && h_nbig == 0 && p->pos_bytes == 1;
    if (fused) {
        if (p->n_own > 0)
            k_compact_lists<<<blocks, kWarpsPerBlock * 32, 0, s>>>(p->adj_ptr.as<int64_t>(), scratch.as<int32_t>(),
                                                                   p->npe, p->n_own, p->nptr.as<int64_t>(),
                                                                   p->ncol.as<int32_t>());
        FEA_CK(cudaGetLastError());
        tr.mark("list compaction", s);
    } else {
        if (p->n_own > 0)
            k_node_pattern<true><<<blocks, kWarpsPerBlock * 32, 0, s>>>(
                p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe,
                p->n_own, nullptr, p->nptr.as<int64_t>(), p->ncol.as<int32_t>(), big.as<int32_t>(),
                nbig.as<unsigned>(), maxbig.as<unsigned>());
        if (h_nbig > 0)
            k_node_pattern_big<true><<<h_nbig, 256, big_smem, s>>>(
                p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe,
                big.as<int32_t>(), nullptr, p->nptr.as<int64_t>(), p->ncol.as<int32_t>());
        FEA_CK(cudaGetLastError());
        tr.mark("node pattern (fill)", s);
        // slot map (adjacency order)
        p->posA.alloc(p->n_adj * p->pstride * p->pos_bytes + 64);
        FEA_CK(cudaMemsetAsync(p->posA.p, 0, p->posA.bytes, s));
        if (p->n_own > 0) {
            if (p->pos_bytes == 1)
                k_pos_adj<uint8_t><<<blocks, kWarpsPerBlock * 32, 0, s>>>(
                    p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe,
                    p->n_own, p->nptr.as<int64_t>(), p->ncol.as<int32_t>(), p->pstride, p->posA.as<uint8_t>());
            else
                k_pos_adj<uint16_t><<<blocks, kWarpsPerBlock * 32, 0, s>>>(
                    p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe,
                    p->n_own, p->nptr.as<int64_t>(), p->ncol.as<int32_t>(), p->pstride, p->posA.as<uint16_t>());
            FEA_CK(cudaGetLastError());
        }
    }
    scratch.reset();
    tr.mark("slot map", s);
    build_runs(p, s);
    tr.mark("CRAC runs", s);
    build_node_order(p, s);
    tr.mark("node order", s);
    build_traversal(p, s);
    tr.mark("traversal records", s);
}

// Common front end: DOFs -> node connectivity (with node-layout detection),
// kept elements, K-row mapping.
void build_elements(fea_plan* p, const int64_t* elem_dofs, int32_t d_hint, cudaStream_t s) {
    DevBuf hold;
    const int64_t* ddofs = device_dofs(elem_dofs, p->E_in * p->m, hold, s);
    DevBuf flags;
    flags.alloc(4);
    DevBuf conn_all;
    int d = (d_hint > 1 && p->m % d_hint == 0) ? d_hint : 1;
    for (;;) {
        const int npe = p->m / d;
        FEA_CK(cudaMemsetAsync(flags.p, 0, 4, s));
        conn_all.alloc(p->E_in * npe * 4);
        if (p->E_in > 0) {
            k_extract_conn<<<grid_for(p->E_in * npe, 256), 256, 0, s>>>(
                ddofs, p->E_in * npe, p->m, d, npe, p->n_rows, conn_all.as<int32_t>(),
                flags.as<unsigned>());
            FEA_CK(cudaGetLastError());
        }
        unsigned h = 0;
        FEA_CK(cudaMemcpyAsync(&h, flags.p, 4, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        FEA_REQUIRE(!(h & 2u), FEA_ERR_INVALID, "element DOF outside [0, n_rows)");
        if ((h & 1u) && d > 1) {
            d = 1;  // not node-contiguous: DOF-level plan
            continue;
        }
        p->d = d;
        p->npe = npe;
        p->dup_nodes = (h & 4u) != 0;
        break;
    }
    FEA_REQUIRE(p->row_begin % p->d == 0 && p->row_end % p->d == 0, FEA_ERR_INVALID,
                "row range must align to node boundaries (multiples of dofs_per_node)");
    const int64_t n_nodes = p->n_rows / p->d;
    FEA_REQUIRE(n_nodes < (int64_t{1} << 31) - 1, FEA_ERR_INVALID, "more than 2^31 nodes");
    p->node_begin = p->row_begin / p->d;
    p->node_end = p->row_end / p->d;
    p->n_own = p->node_end - p->node_begin;
    p->partitioned = !(p->row_begin == 0 && p->row_end == p->n_rows);
    if (!p->partitioned) {
        p->E = p->E_in;
        p->elem_id.alloc(p->E * 8);
        if (p->E > 0) k_iota64<<<grid_for(p->E, 256), 256, 0, s>>>(p->elem_id.as<int64_t>(), p->E);
        p->conn_k = std::move(conn_all);
    } else {
        DevBuf keep, pos;
        keep.alloc((p->E_in + 1) * 8);
        pos.alloc((p->E_in + 1) * 8);
        FEA_CK(cudaMemsetAsync(keep.p, 0, keep.bytes, s));
        if (p->E_in > 0)
            k_keep_flags<<<grid_for(p->E_in, 256), 256, 0, s>>>(
                conn_all.as<int32_t>(), p->E_in, p->npe, p->node_begin, p->node_end,
                keep.as<int64_t>());
        exclusive_sum(keep.as<int64_t>(), pos.as<int64_t>(), p->E_in + 1, s);
        FEA_CK(cudaMemcpyAsync(&p->E, pos.as<int64_t>() + p->E_in, 8, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        p->elem_id.alloc(p->E * 8);
        if (p->E_in > 0)
            k_scatter_kept<<<grid_for(p->E_in, 256), 256, 0, s>>>(keep.as<int64_t>(),
                                                                  pos.as<int64_t>(), p->E_in,
                                                                  p->elem_id.as<int64_t>());
        if (p->k_compact) {
            p->conn_k.alloc(p->E * p->npe * 4);
            if (p->E > 0)
                k_gather_conn<<<grid_for(p->E * p->npe, 256), 256, 0, s>>>(
                    conn_all.as<int32_t>(), p->elem_id.as<int64_t>(), p->E, p->npe,
                    p->conn_k.as<int32_t>());
        } else {
            p->conn_k = std::move(conn_all);
        }
    }
    FEA_CK(cudaGetLastError());
    p->elem_krow.alloc(p->E * 4);
    if (p->E > 0)
        k_krow<<<grid_for(p->E, 256), 256, 0, s>>>(p->elem_id.as<int64_t>(), p->E,
                                                   p->k_compact || !p->partitioned,
                                                   p->elem_krow.as<int32_t>());
    FEA_CK(cudaGetLastError());
}

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { FEA_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        if (s) cudaStreamDestroy(s);
    }
};

template <class F>
fea_status guarded(F&& f) {
    try {
        g_err.clear();
        f();
        return FEA_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return FEA_ERR_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FEA_ERR_INVALID;
    }
}

// Copy n bytes from a device buffer to a host-or-device destination.
void copy_out(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (n == 0) return;
    FEA_CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, s));
}

// Host-side conn of the kept elements, in ascending element id.
std::vector<int32_t> host_conn(const fea_plan* p, cudaStream_t s) {
    std::vector<int32_t> h(static_cast<size_t>(p->E * p->npe));
    std::vector<int32_t> kr(static_cast<size_t>(p->E));
    if (p->E == 0) return h;
    std::vector<int32_t> all(static_cast<size_t>(p->krows() * p->npe));
    FEA_CK(cudaMemcpyAsync(all.data(), p->conn_k.p, all.size() * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(kr.data(), p->elem_krow.p, kr.size() * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    for (int64_t e = 0; e < p->E; ++e)
        std::memcpy(&h[e * p->npe], &all[static_cast<size_t>(kr[e]) * p->npe], p->npe * 4);
    return h;
}

// Per-node incidences in ascending (colour, element id) plus their position rows.
void build_colour_incidences(fea_plan* p, const DevBuf& d_ck, int nc, cudaStream_t s) {
    const int64_t n = p->n_adj;
    const int row_bytes = p->pstride * p->pos_bytes;
    p->adjC.alloc(n * 4 + 64);
    p->posAC.alloc(n * row_bytes + 64);
    FEA_CK(cudaMemsetAsync(p->posAC.p, 0, p->posAC.bytes, s));
    if (n == 0) return;
    DevBuf node_of, k1, v1, k2, v2;
    node_of.alloc(n * 4);
    k1.alloc(n * 4); v1.alloc(n * 4); k2.alloc(n * 4); v2.alloc(n * 4);
    k_node_of<<<grid_for(p->n_own, 256), 256, 0, s>>>(p->adj_ptr.as<int64_t>(), p->n_own, node_of.as<int32_t>());
    k_colour_keys<<<grid_for(n, 256), 256, 0, s>>>(p->adj.as<int32_t>(), n, p->npe, d_ck.as<int32_t>(),
                                                   k1.as<uint32_t>(), v1.as<int32_t>());
    FEA_CK(cudaGetLastError());
    // pass 1: stable by colour
    radix_sort_pairs(k1.as<uint32_t>(), k2.as<uint32_t>(), v1.as<int32_t>(), v2.as<int32_t>(), n, 0,
                     bits_for(static_cast<uint64_t>(nc)), s);
    k_gather_keys<<<grid_for(n, 256), 256, 0, s>>>(node_of.as<int32_t>(), v2.as<int32_t>(), n, k1.as<uint32_t>());
    FEA_CK(cudaGetLastError());
    // pass 2: stable by node
    radix_sort_pairs(k1.as<uint32_t>(), k2.as<uint32_t>(), v2.as<int32_t>(), v1.as<int32_t>(), n, 0,
                     bits_for(static_cast<uint64_t>(p->n_own)), s);
    k_permute_incidences<<<grid_for(n, 256), 256, 0, s>>>(v1.as<int32_t>(), n, row_bytes, p->adj.as<int32_t>(),
                                                          p->posA.as<unsigned char>(), p->adjC.as<int32_t>(),
                                                          p->posAC.as<unsigned char>());
    FEA_CK(cudaGetLastError());
    // d = 1 with traversal records: the colour-ordered incidences get their own records (same
    // per-node counts and offsets, trav_ptr / trav_meta), so FEA_DET_COLOUR reads them
    // sequentially like the sorted route
    p->trav_recC.reset();
    p->cnr_recC.reset();
    p->slot_recC.reset();
    if (p->trav_rec.p) {
        const int pw = p->pstride * p->pos_bytes / 4;
        p->trav_recC.alloc(std::max<int64_t>(n, 1) * p->trav_rw * 4);
        k_trav_records<<<grid_for(p->n_own * 32, 256), 256, 0, s>>>(
            p->node_order.as<int32_t>(), p->adj_ptr.as<int64_t>(), p->adjC.as<int32_t>(),
            static_cast<const uint32_t*>(p->posAC.p), pw, p->trav_rw, p->trav_ptr.as<int64_t>(), p->n_own,
            p->trav_recC.as<int32_t>());
        FEA_CK(cudaGetLastError());
        build_lane_records(p, p->trav_recC, p->ln_recC, s);
    }
    FEA_CK(cudaStreamSynchronize(s));
}

}  // namespace

int64_t metadata_bytes(const fea_plan* p) {
    return static_cast<int64_t>(p->conn_k.bytes + p->elem_id.bytes + p->elem_krow.bytes +
                                p->adj_ptr.bytes + p->adj.bytes + p->nptr.bytes + p->ncol.bytes +
                                p->nrun_ptr.bytes + p->posA.bytes + p->posE.bytes +
                                p->order.bytes + p->at_krow.bytes + p->at_rows.bytes + p->at_pos.bytes + p->colour_elems.bytes + p->adjC.bytes + p->posAC.bytes +
                                p->node_order.bytes + p->trav_ptr.bytes + p->trav_meta.bytes +
                                p->trav_rec.bytes + p->trav_recC.bytes + p->ln_slot.bytes + p->ln_hdr.bytes +
                                p->ln_rec.bytes + p->ln_recC.bytes + p->cnr_hdr.bytes + p->cnr_rec.bytes +
                                p->cnr_recC.bytes + p->slot_hdr.bytes + p->slot_rec.bytes + p->slot_recC.bytes +
                                p->pk_hdr.bytes + p->pk_krow.bytes + p->pk_cidx.bytes + p->pk_rows.bytes + p->pk_rowpair.bytes +
                                p->pk_pairs.bytes + p->sk_meta.bytes + p->sk_shape.bytes + p->sk_k0.bytes + p->sk_krow.bytes);
}

}  // namespace feagpu

int64_t fea_plan::kbytes_required() const { return krows() * static_cast<int64_t>(m) * m * 8; }

using namespace feagpu;

extern "C" {

const char* fea_last_error(void) { return g_err.c_str(); }

int fea_version(void) { return 100; }

fea_status fea_plan_create(int device, const int64_t* elem_dofs, int64_t n_elements, int32_t m,
                           int64_t n_rows, int32_t dofs_per_node, int64_t row_begin,
                           int64_t row_end, uint32_t flags, fea_plan** out) {
    return guarded([&] {
        FEA_REQUIRE(out, FEA_ERR_INVALID, "out is NULL");
        *out = nullptr;
        FEA_REQUIRE(n_elements >= 0 && m >= 1 && n_rows >= 0, FEA_ERR_INVALID,
                    "need n_elements >= 0, m >= 1, n_rows >= 0");
        FEA_REQUIRE(n_elements == 0 || elem_dofs, FEA_ERR_INVALID, "elem_dofs is NULL");
        FEA_REQUIRE(dofs_per_node >= 1, FEA_ERR_INVALID, "dofs_per_node must be >= 1");
        FEA_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= n_rows, FEA_ERR_INVALID,
                    "row range must satisfy 0 <= row_begin <= row_end <= n_rows");
        DeviceScope ds(device);
        Stream st;
        auto p = std::make_unique<fea_plan>();
        p->device = device;
        FEA_CK(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device));
        p->kn = read_knobs();
        p->cn_disabled = std::getenv("FEA_GATHER_NO_CN") != nullptr;
        p->d1_disabled = std::getenv("FEA_GATHER_NO_D1") != nullptr;
        p->slot_disabled = std::getenv("FEA_GATHER_NO_SLOT") != nullptr;
        p->E_in = n_elements;
        p->m = m;
        p->n_rows = n_rows;
        p->row_begin = row_begin;
        p->row_end = row_end;
        p->k_compact = (flags & FEA_PLAN_K_COMPACT) != 0;
        StageTrace tr;
        build_elements(p.get(), elem_dofs, dofs_per_node, st.s);
        tr.mark("DOFs -> connectivity", st.s);
        build_adjacency(p.get(), st.s);
        tr.mark("incidences sort + scan", st.s);
        build_own_pattern(p.get(), st.s);
        FEA_CK(cudaStreamSynchronize(st.s));
        *out = p.release();
    });
}

fea_status fea_plan_create_with_pattern(int device, const int64_t* elem_dofs, int64_t n_elements,
                                        int32_t m, int64_t n_rows, int32_t format,
                                        const int64_t* row_ptr, const int64_t* idx,
                                        fea_plan** out) {
    return guarded([&] {
        FEA_REQUIRE(out, FEA_ERR_INVALID, "out is NULL");
        *out = nullptr;
        FEA_REQUIRE(format == FEA_FORMAT_CSR || format == FEA_FORMAT_CRAC, FEA_ERR_INVALID,
                    "unknown pattern format");
        FEA_REQUIRE(n_elements >= 0 && m >= 1 && n_rows >= 0 && row_ptr && (n_rows == 0 || idx),
                    FEA_ERR_INVALID, "bad arguments");
        FEA_REQUIRE(n_rows < (int64_t{1} << 31) - 1, FEA_ERR_INVALID, "more than 2^31 rows");
        DeviceScope ds(device);
        Stream st;
        cudaStream_t s = st.s;
        // The caller's arrays (host, like the reference's, or device) are validated and turned
        // into the plan's layout on the device: nothing here is O(nnz) on the host.
        const bool crac = format == FEA_FORMAT_CRAC;
        FEA_REQUIRE(!crac || idx, FEA_ERR_INVALID, "a CRAC pattern needs its col_align array (at least (0, 0))");
        int64_t first = 0, last = 0;
        FEA_CK(cudaMemcpy(&first, row_ptr, 8, cudaMemcpyDefault));
        FEA_CK(cudaMemcpy(&last, row_ptr + n_rows, 8, cudaMemcpyDefault));
        FEA_REQUIRE(first == 0, FEA_ERR_INVALID, "row_ptr[0] must be 0");
        FEA_REQUIRE(last >= 0, FEA_ERR_INVALID, "row_ptr not monotone");
        FEA_REQUIRE(last <= (int64_t{1} << 40), FEA_ERR_INVALID, "row_ptr[n_rows] out of range");
        DevBuf hold_ptr, hold_idx, d_err, d_max;
        auto on_device = [&](const int64_t* src, int64_t n, DevBuf& hold) -> const int64_t* {
            if (n == 0 || is_device_ptr(src)) return src;
            hold.alloc(static_cast<size_t>(n) * 8);
            FEA_CK(cudaMemcpyAsync(hold.p, src, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s));
            return hold.as<int64_t>();
        };
        const int64_t* in_ptr = on_device(row_ptr, n_rows + 1, hold_ptr);
        d_err.alloc(4);
        d_max.alloc(8);
        FEA_CK(cudaMemsetAsync(d_err.p, 0xff, 4, s));
        FEA_CK(cudaMemsetAsync(d_max.p, 0, 8, s));
        auto check = [&] {
            unsigned h = kExtOk;
            FEA_CK(cudaGetLastError());
            FEA_CK(cudaMemcpyAsync(&h, d_err.p, 4, cudaMemcpyDeviceToHost, s));
            FEA_CK(cudaStreamSynchronize(s));
            FEA_REQUIRE(h == kExtOk, FEA_ERR_INVALID, ext_err_text(h));
        };
        k_ext_check_ptr<<<grid_for(n_rows + 1, 256), 256, 0, s>>>(in_ptr, n_rows, crac, d_err.as<unsigned>());
        check();  // the row pointers are safe to index with from here on
        // CSR view: d_ptr / d_cols (the caller's own arrays for a CSR pattern)
        DevBuf own_ptr, own_cols, miss;
        const int64_t* d_ptr = in_ptr;
        const int64_t* d_cols = nullptr;
        const int64_t* d_cptr = nullptr;
        const int64_t* d_align = nullptr;
        int64_t nnz = last;
        if (!crac) {
            d_cols = on_device(idx, nnz, hold_idx);
        } else {
            const int64_t n_align = last + 2;
            d_cptr = in_ptr;
            d_align = on_device(idx, n_align, hold_idx);
            k_ext_check_runs<<<grid_for(n_align / 2, 256), 256, 0, s>>>(d_align, n_align, n_rows,
                                                                        d_err.as<unsigned>());
            check();
            FEA_CK(cudaMemcpy(&nnz, d_align + n_align - 1, 8, cudaMemcpyDefault));
            FEA_REQUIRE(nnz >= 0 && nnz <= (int64_t{1} << 40), FEA_ERR_INVALID, "CRAC nnz out of range");
            own_ptr.alloc((n_rows + 1) * 8);
            own_cols.alloc(static_cast<size_t>(nnz) * 8);
            k_ext_crac_csr_ptr<<<grid_for(n_rows + 1, 256), 256, 0, s>>>(d_cptr, d_align, n_rows,
                                                                         own_ptr.as<int64_t>());
            k_ext_crac_cols<<<grid_for((n_align - 2) / 2 * 32, 256), 256, 0, s>>>(d_align, (n_align - 2) / 2,
                                                                                   own_cols.as<int64_t>());
            d_ptr = own_ptr.as<int64_t>();
            d_cols = own_cols.as<int64_t>();
        }
        auto p = std::make_unique<fea_plan>();
        p->device = device;
        FEA_CK(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device));
        p->kn = read_knobs();
        p->external = true;
        p->E_in = n_elements;
        p->m = m;
        p->n_rows = n_rows;
        p->row_begin = 0;
        p->row_end = n_rows;
        // node-level pattern == the caller's pattern (d = 1)
        p->nptr.alloc((n_rows + 1) * 8);
        FEA_CK(cudaMemcpyAsync(p->nptr.p, d_ptr, (n_rows + 1) * 8, cudaMemcpyDeviceToDevice, s));
        p->ncol.alloc(static_cast<size_t>(nnz) * 4);
        if (n_rows > 0)
            k_ext_check_rows<<<grid_for(n_rows * 32, 256), 256, 0, s>>>(
                d_ptr, d_cols, n_rows, p->ncol.as<int32_t>(), d_err.as<unsigned>(),
                d_max.as<unsigned long long>());
        check();
        unsigned long long max_len = 0;
        FEA_CK(cudaMemcpy(&max_len, d_max.p, 8, cudaMemcpyDeviceToHost));
        FEA_REQUIRE(max_len <= 65536, FEA_ERR_INVALID, "pattern row longer than 65536 entries");
        build_elements(p.get(), elem_dofs, 1, s);
        build_adjacency(p.get(), s);
        p->max_cnt = static_cast<int32_t>(max_len);
        p->pos_bytes = max_len <= 256 ? 1 : 2;
        p->pstride = ((p->npe * p->pos_bytes + 3) / 4 * 4) / p->pos_bytes;
        p->nnz_nodes = nnz;
        p->nnz = nnz;
        miss.alloc(8);
        FEA_CK(cudaMemsetAsync(miss.p, 0xff, 8, s));
        p->posA.alloc(p->n_adj * p->pstride * p->pos_bytes + 64);
        FEA_CK(cudaMemsetAsync(p->posA.p, 0, p->posA.bytes, s));
        const unsigned blocks = grid_for(n_rows * 32, 256);
        if (n_rows > 0) {
#define FEA_LAUNCH_EXT(T, C)                                                                   \
    k_pos_external<T, C><<<blocks, 256, 0, s>>>(                                               \
        p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), p->conn_k.as<int32_t>(), p->npe, n_rows, \
        d_ptr, d_cols, d_cptr, d_align, p->pstride, p->posA.as<T>(), miss.as<unsigned long long>())
            if (p->pos_bytes == 1) {
                if (crac) FEA_LAUNCH_EXT(uint8_t, true); else FEA_LAUNCH_EXT(uint8_t, false);
            } else {
                if (crac) FEA_LAUNCH_EXT(uint16_t, true); else FEA_LAUNCH_EXT(uint16_t, false);
            }
#undef FEA_LAUNCH_EXT
            FEA_CK(cudaGetLastError());
        }
        unsigned long long hm = 0;
        FEA_CK(cudaMemcpyAsync(&hm, miss.p, 8, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        if (hm != ~0ull) {
            const int64_t mm = static_cast<int64_t>(p->m) * p->m;
            const int64_t e = static_cast<int64_t>(hm) / mm;
            const int64_t rem = static_cast<int64_t>(hm) - e * mm;
            const int a = static_cast<int>(rem / p->m), b = static_cast<int>(rem % p->m);
            std::vector<int64_t> hd(static_cast<size_t>(p->m));
            FEA_CK(cudaMemcpy(hd.data(), elem_dofs + e * p->m, p->m * 8, cudaMemcpyDefault));
            p->miss_e = e;
            p->miss_r = hd[a];
            p->miss_c = hd[b];
        }
        build_runs(p.get(), s);
        build_node_order(p.get(), s);
        build_traversal(p.get(), s);
        FEA_CK(cudaStreamSynchronize(s));
        *out = p.release();
    });
}

void fea_plan_destroy(fea_plan* plan) {
    if (!plan) return;
    try {
        DeviceScope ds(plan->device);
        delete plan;
    } catch (...) {
        delete plan;
    }
}

fea_status fea_plan_sizes(const fea_plan* p, int64_t* n_rows, int64_t* nnz, int64_t* n_runs,
                          int64_t* n_elements) {
    return guarded([&] {
        FEA_REQUIRE(p, FEA_ERR_INVALID, "plan is NULL");
        if (n_rows) *n_rows = p->n_own * p->d;
        if (nnz) *nnz = p->nnz;
        if (n_runs) *n_runs = p->n_runs;
        if (n_elements) *n_elements = p->E;
    });
}

fea_status fea_plan_info(const fea_plan* p, int32_t* dofs_per_node, int32_t* nodes_per_element,
                         int64_t* meta) {
    return guarded([&] {
        FEA_REQUIRE(p, FEA_ERR_INVALID, "plan is NULL");
        if (dofs_per_node) *dofs_per_node = p->d;
        if (nodes_per_element) *nodes_per_element = p->npe;
        if (meta) *meta = metadata_bytes(p);
    });
}

// Device destinations are written in place (config 5's cols are 32.7 GB: no device temp);
// cols / col_align may be NULL to fetch only the row pointers.
fea_status fea_plan_copy_csr(const fea_plan* p, int64_t* row_ptr, int64_t* cols) {
    return guarded([&] {
        FEA_REQUIRE(p && row_ptr, FEA_ERR_INVALID, "NULL argument");
        DeviceScope ds(p->device);
        Stream st;
        const int64_t rows = p->n_own * p->d;
        DevBuf drp, dcols;
        int64_t* rp_d = row_ptr;
        int64_t* cols_d = cols;
        if (!is_device_ptr(row_ptr)) {
            drp.alloc((rows + 1) * 8);
            rp_d = drp.as<int64_t>();
        }
        if (cols && !is_device_ptr(cols)) {
            dcols.alloc(p->nnz * 8);
            cols_d = dcols.as<int64_t>();
        }
        FEA_CK(cudaMemsetAsync(rp_d, 0, 8, st.s));
        if (p->n_own > 0)
            k_expand_csr<<<grid_for(p->n_own * 32, 256), 256, 0, st.s>>>(
                p->nptr.as<int64_t>(), p->ncol.as<int32_t>(), p->n_own, p->d, p->node_begin, rp_d, cols_d);
        FEA_CK(cudaGetLastError());
        if (drp.p) copy_out(row_ptr, drp.p, (rows + 1) * 8, st.s);
        if (dcols.p) copy_out(cols, dcols.p, p->nnz * 8, st.s);
        FEA_CK(cudaStreamSynchronize(st.s));
    });
}

fea_status fea_plan_copy_crac(const fea_plan* p, int64_t* row_ptr, int64_t* col_align) {
    return guarded([&] {
        FEA_REQUIRE(p && row_ptr, FEA_ERR_INVALID, "NULL argument");
        DeviceScope ds(p->device);
        Stream st;
        const int64_t rows = p->n_own * p->d;
        DevBuf dptr, dal;
        int64_t* ptr_d = row_ptr;
        int64_t* al_d = col_align;
        if (!is_device_ptr(row_ptr)) {
            dptr.alloc((rows + 1) * 8);
            ptr_d = dptr.as<int64_t>();
        }
        if (!col_align || !is_device_ptr(col_align)) {  // the kernel always writes the pairs
            dal.alloc((2 * p->n_runs + 2) * 8);
            al_d = dal.as<int64_t>();
        }
        if (p->n_own > 0) {
            k_expand_crac<<<grid_for(p->n_own, 128), 128, 0, st.s>>>(
                p->nptr.as<int64_t>(), p->ncol.as<int32_t>(), p->nrun_ptr.as<int64_t>(), p->n_own,
                p->d, ptr_d, al_d);
            FEA_CK(cudaGetLastError());
        } else {
            const int64_t z[2] = {0, 0};
            FEA_CK(cudaMemcpyAsync(ptr_d, z, 8, cudaMemcpyHostToDevice, st.s));
            FEA_CK(cudaMemcpyAsync(al_d, z, 16, cudaMemcpyHostToDevice, st.s));
        }
        if (dptr.p) copy_out(row_ptr, dptr.p, (rows + 1) * 8, st.s);
        if (col_align && dal.p) copy_out(col_align, dal.p, (2 * p->n_runs + 2) * 8, st.s);
        FEA_CK(cudaStreamSynchronize(st.s));
    });
}

fea_status fea_plan_copy_elements(const fea_plan* p, int64_t* elem_ids) {
    return guarded([&] {
        FEA_REQUIRE(p && (p->E == 0 || elem_ids), FEA_ERR_INVALID, "NULL argument");
        DeviceScope ds(p->device);
        FEA_CK(cudaMemcpy(elem_ids, p->elem_id.p, p->E * 8, cudaMemcpyDefault));
    });
}

// greedy_colouring (colouring.cpp:24-75) over the plan's elements in ascending
// id. Inherently sequential (each element depends on all earlier ones): host.
fea_status fea_plan_greedy_colouring(const fea_plan* p, int32_t* colour_of, int32_t* n_colours) {
    return guarded([&] {
        FEA_REQUIRE(p && (p->E == 0 || colour_of), FEA_ERR_INVALID, "NULL argument");
        DeviceScope ds(p->device);
        Stream st;
        const std::vector<int32_t> conn = host_conn(p, st.s);
        const int npe = p->npe;
        int64_t n_nodes = 0;
        for (const int32_t v : conn) n_nodes = std::max<int64_t>(n_nodes, v + 1);
        std::vector<int64_t> ptr(static_cast<size_t>(n_nodes) + 1, 0);
        for (const int32_t v : conn) ++ptr[v + 1];
        for (int64_t v = 0; v < n_nodes; ++v) ptr[v + 1] += ptr[v];
        std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
        std::vector<int32_t> adj(conn.size());
        for (int64_t e = 0; e < p->E; ++e)
            for (int a = 0; a < npe; ++a) adj[fill[conn[e * npe + a]]++] = static_cast<int32_t>(e);
        std::vector<int32_t> col(static_cast<size_t>(p->E), -1);
        std::vector<char> used;
        int nc = 0;
        for (int64_t e = 0; e < p->E; ++e) {
            std::fill(used.begin(), used.end(), 0);
            for (int a = 0; a < npe; ++a) {
                const int32_t v = conn[e * npe + a];
                for (int64_t k = ptr[v]; k < ptr[v + 1] && adj[k] < e; ++k) {  // (ascending: only earlier elements are coloured)
                    const int c = col[adj[k]];
                    if (static_cast<size_t>(c) >= used.size()) used.resize(c + 1, 0);
                    used[c] = 1;
                }
            }
            int c = 0;
            while (static_cast<size_t>(c) < used.size() && used[c]) ++c;
            col[e] = c;
            nc = std::max(nc, c + 1);
        }
        std::memcpy(colour_of, col.data(), col.size() * 4);
        if (n_colours) *n_colours = nc;
    });
}

fea_status fea_plan_set_colouring(fea_plan* p, const int32_t* colour_of) {
    return guarded([&] {
        FEA_REQUIRE(p && (p->E == 0 || colour_of), FEA_ERR_INVALID, "NULL argument");
        DeviceScope ds(p->device);
        Stream st;
        std::vector<int32_t> col(static_cast<size_t>(p->E));
        if (p->E > 0) FEA_CK(cudaMemcpy(col.data(), colour_of, col.size() * 4, cudaMemcpyDefault));
        int nc = 0;
        for (const int32_t c : col) {
            FEA_REQUIRE(c >= 0, FEA_ERR_INVALID, "negative colour");
            nc = std::max(nc, c + 1);
        }
        // colour of every K row on the device, and the conflict question answered there (a node
        // with two different incident elements of one colour); only an invalid colouring takes
        // the host scan below, which names the pair the reference's scan would name
        DevBuf d_col, d_ck, d_flag;
        d_col.alloc(std::max<size_t>(col.size(), 1) * 4);
        d_ck.alloc(std::max<int64_t>(p->krows(), 1) * 4);
        d_flag.alloc(4);
        FEA_CK(cudaMemsetAsync(d_ck.p, 0, d_ck.bytes, st.s));
        FEA_CK(cudaMemsetAsync(d_flag.p, 0, 4, st.s));
        unsigned conflict = 0;
        if (p->E > 0) {
            FEA_CK(cudaMemcpyAsync(d_col.p, col.data(), col.size() * 4, cudaMemcpyHostToDevice, st.s));
            k_colour_of_krow<<<grid_for(p->E, 256), 256, 0, st.s>>>(p->elem_krow.as<int32_t>(), d_col.as<int32_t>(), p->E,
                                                                   d_ck.as<int32_t>());
            if (p->n_own > 0)
                k_colour_conflict<<<grid_for(p->n_own, 128), 128, 0, st.s>>>(p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(),
                                                                            p->n_own, p->npe, d_ck.as<int32_t>(),
                                                                            d_flag.as<unsigned>());
            FEA_CK(cudaGetLastError());
            FEA_CK(cudaMemcpyAsync(&conflict, d_flag.p, 4, cudaMemcpyDeviceToHost, st.s));
            FEA_CK(cudaStreamSynchronize(st.s));
        }
        const int npe = p->npe;
        std::vector<int64_t> off(static_cast<size_t>(nc) + 1, 0);
        for (const int32_t c : col) ++off[c + 1];
        for (int c = 0; c < nc; ++c) off[c + 1] += off[c];
        std::vector<int32_t> by_colour(col.size());
        {
            std::vector<int64_t> f(off.begin(), off.end() - 1);
            for (int64_t e = 0; e < p->E; ++e) by_colour[f[col[e]]++] = static_cast<int32_t>(e);
        }
        if (conflict) {
            // find_colour_conflict (colouring.cpp:91-119): same-colour elements may
            // not share a DOF; with node-contiguous DOFs that is sharing a node.
            const std::vector<int32_t> conn = host_conn(p, st.s);
            int64_t n_nodes = 0;
            for (const int32_t v : conn) n_nodes = std::max<int64_t>(n_nodes, v + 1);
            std::vector<int64_t> owner(static_cast<size_t>(n_nodes), -1);
            for (int c = 0; c < nc; ++c) {
                for (int64_t i = off[c]; i < off[c + 1]; ++i) {
                    const int32_t e = by_colour[i];
                    for (int a = 0; a < npe; ++a) {
                        const int32_t v = conn[static_cast<int64_t>(e) * npe + a];
                        // only owned rows are assembled: sharing a node outside them is no conflict
                        if (v < p->node_begin || v >= p->node_end) continue;
                        if (owner[v] >= 0 && owner[v] != e)
                            throw Error(FEA_ERR_INVALID_COLOURING,
                                        "invalid colouring: elements " + std::to_string(owner[v]) +
                                            " and " + std::to_string(e) + " share dof " +
                                            std::to_string(static_cast<int64_t>(v) * p->d) +
                                            " within one colour");
                        owner[v] = e;
                    }
                }
                for (int64_t i = off[c]; i < off[c + 1]; ++i)
                    for (int a = 0; a < npe; ++a) {
                        const int32_t v = conn[static_cast<int64_t>(by_colour[i]) * npe + a];
                        if (v >= p->node_begin && v < p->node_end) owner[v] = -1;
                    }
            }
            throw Error(FEA_ERR_INVALID_COLOURING, "invalid colouring: two elements of one colour share a dof");
        }
        p->colour_elems.alloc(by_colour.size() * 4);
        if (!by_colour.empty())
            FEA_CK(cudaMemcpy(p->colour_elems.p, by_colour.data(), by_colour.size() * 4,
                              cudaMemcpyHostToDevice));
        p->colour_off = off;
        build_colour_incidences(p, d_ck, std::max(nc, 1), st.s);
        p->has_colouring = true;
    });
}

// Jones-Plassmann colouring on the device (a valid colouring, not the greedy one; the colour
// routes stay bit-identical to assemble_coloured_vectorized under whichever colouring is set).
fea_status fea_plan_jp_colouring(const fea_plan* p, uint64_t seed, int32_t* colour_of, int32_t* n_colours) {
    return guarded([&] {
        FEA_REQUIRE(p && (p->E == 0 || colour_of), FEA_ERR_INVALID, "NULL argument");
        DeviceScope ds(p->device);
        Stream st;
        cudaStream_t s = st.s;
        if (p->E == 0) {
            if (n_colours) *n_colours = 0;
            return;
        }
        DevBuf prio, col, rem, k2l;
        prio.alloc(p->E * 8);
        col.alloc(p->E * 4);
        rem.alloc(8);
        const int32_t* k2l_ptr = nullptr;
        if (p->partitioned && !p->k_compact) {  // adjacency holds global element ids
            k2l.alloc(p->E_in * 4);
            FEA_CK(cudaMemsetAsync(k2l.p, 0xff, k2l.bytes, s));
            std::vector<int32_t> kr(static_cast<size_t>(p->E)), inv(static_cast<size_t>(p->E_in), -1);
            FEA_CK(cudaMemcpy(kr.data(), p->elem_krow.p, kr.size() * 4, cudaMemcpyDeviceToHost));
            for (int64_t le = 0; le < p->E; ++le) inv[kr[le]] = static_cast<int32_t>(le);
            FEA_CK(cudaMemcpyAsync(k2l.p, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice, s));
            k2l_ptr = k2l.as<int32_t>();
        }
        k_jp_prio<<<grid_for(p->E, 256), 256, 0, s>>>(p->elem_id.as<int64_t>(), p->E, seed,
                                                      prio.as<uint64_t>(), col.as<int32_t>());
        FEA_CK(cudaGetLastError());
        for (int round = 0; round < 100000; ++round) {
            FEA_CK(cudaMemsetAsync(rem.p, 0, 8, s));
            k_jp_round<<<grid_for(p->E, 256), 256, 0, s>>>(
                p->conn_k.as<int32_t>(), p->elem_krow.as<int32_t>(), k2l_ptr, p->E, p->npe, p->node_begin,
                p->node_end, p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(), prio.as<uint64_t>(),
                col.as<int32_t>(), rem.as<unsigned long long>());
            FEA_CK(cudaGetLastError());
            unsigned long long h = 0;
            FEA_CK(cudaMemcpyAsync(&h, rem.p, 8, cudaMemcpyDeviceToHost, s));
            FEA_CK(cudaStreamSynchronize(s));
            if (h == 0) break;
        }
        std::vector<int32_t> hc(static_cast<size_t>(p->E));
        FEA_CK(cudaMemcpy(hc.data(), col.p, hc.size() * 4, cudaMemcpyDeviceToHost));
        int nc = 0;
        for (const int32_t c : hc) {
            FEA_REQUIRE(c >= 0 && c < 128, FEA_ERR_INVALID, "Jones-Plassmann colouring needs more than 128 colours");
            nc = std::max(nc, c + 1);
        }
        std::memcpy(colour_of, hc.data(), hc.size() * 4);
        if (n_colours) *n_colours = nc;
    });
}

fea_status fea_plan_missing_entry(const fea_plan* p, int64_t* element, int64_t* row, int64_t* col) {
    return guarded([&] {
        FEA_REQUIRE(p, FEA_ERR_INVALID, "plan is NULL");
        if (element) *element = p->miss_e;
        if (row) *row = p->miss_r;
        if (col) *col = p->miss_c;
    });
}

int32_t fea_plan_last_launches(const fea_plan* p) { return p ? p->last_launches : 0; }

}  // extern "C"
