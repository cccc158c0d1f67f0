// Kernels and their launchers for the numeric phase (included by numeric.cu and by the
// position-type instantiation units gather_u8.cu / gather_u16.cu; everything here is
// TU-local, see numeric.cu for the design notes of every kernel).
#pragma once

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.cuh"
#include "prims.cuh"

namespace feagpu {
extern thread_local std::string g_err;

namespace {

constexpr int kWarps = 4;  // warps per CTA for the numeric kernels



// lazily built plan tables are allocated on first use; inside a stream capture (CUDA graph)
// allocation is not allowed, so the kernels that read them fall back to the table-free path
bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 64) b = 148 * 64;
    return static_cast<unsigned>(b);
}

__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }

// Debug builds (-DFEA_DEBUG, tools/sanitize_case.py): trap on any out-of-range index.
#ifdef FEA_DEBUG
#define FEA_DCHECK(cond)     \
    do {                     \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define FEA_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

// Seeded element-matrix generator (the counter-hash supplier): the same bits
// as oracle/oracle.c orc_kval. kgen_elem is hoisted per element, kgen_entry per entry.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t kgen_elem(uint64_t seed, int64_t id) {
    return mix64(seed + static_cast<uint64_t>(id));
}
__device__ __forceinline__ double kgen_entry(uint64_t he, int i, int j) {
    const uint64_t lo = static_cast<uint64_t>(i < j ? i : j);
    const uint64_t hi = static_cast<uint64_t>(i < j ? j : i);
    const uint64_t h = mix64(he ^ ((lo << 32) | hi));
    return static_cast<double>(h >> 11) * 0x1p-53 * 2.0 - 1.0;
}
__device__ __forceinline__ double kval(uint64_t seed, int64_t e, int i, int j) {
    return kgen_entry(kgen_elem(seed, e), i, j);
}

// Fused supplier: when on, the gather kernels generate K[e][i][j] in registers instead of
// reading it (fea_assemble_seeded) — no 8*E*m^2 bytes of K traffic.
// Thrown by a gather launcher whose shared-memory layout cannot hold the plan's largest node
// row block (a hub node with hundreds of neighbours, or d * m > 512): gather() then takes
// k_gather_global, which accumulates in the values array itself.
struct DoesNotFit {};
#define FEA_FITS(cond)                  \
    do {                                \
        if (!(cond)) throw DoesNotFit{}; \
    } while (0)

struct GenK {
    int on;
    uint64_t seed;
    const int64_t* ids;  // element id per K row (nullptr: the K row is the element id)
};

// --- TMA bulk copy + mbarrier primitives (sm_90+/sm_100a PTX) ---------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
}
// 1D bulk copy global -> shared (TMA, SASS UBLKCP), completion via mbarrier tx bytes;
// L2 evict-first: each K byte is read exactly once.
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes,
                                            uint32_t bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Ampere-style async copy global -> shared (SASS LDGSTS), 8 or 16 bytes per lane,
// bypassing registers; completion tracked by an mbarrier (cp.async.mbarrier.arrive).
template <int UNIT>
__device__ __forceinline__ void cp_async(uint32_t dst, uint64_t src) {
    if constexpr (UNIT == 16)
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Programmatic dependent launch: a kernel launched with the PDL attribute may start while the
// previous kernel of its stream is still running; it reads only plan metadata (constant for the
// plan) before pdl_wait(), and K / values (which the previous kernel may have written) after.
// Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

#ifndef FEA_GATHER_MIN_BLOCKS
#define FEA_GATHER_MIN_BLOCKS 5
#endif
#ifndef FEA_GATHER_MIN_BLOCKS_WIDE
#define FEA_GATHER_MIN_BLOCKS_WIDE 4
#endif
// ---------------------------------------------------------------------------
// Deterministic owner-computes gather, one node per lane group (FEA_DET_SORTED)
// ---------------------------------------------------------------------------
// A group of G lanes owns one node: the node's d rows are one contiguous block of
// values. The group streams the node's incident element-matrix row blocks
// K[e][a*d..a*d+d-1][:] (d*m contiguous doubles each, one per incident element,
// ascending element id) straight into registers — R rounds of G entries per
// block, PF blocks in flight — and folds them into a shared-memory copy of the
// node block (one __syncwarp between blocks), then writes the block once with
// coalesced streaming stores. Per slot this is a left fold from the slot's
// start value in ascending element order: bit-identical to assemble_sequential
// (assembly.hpp:112-118). K is read once, values written once, no atomics.
// The node's incidence list and position-map slice are loaded once per node
// (coalesced, into registers / shared memory) so no dependent global load sits
// between two row-block loads. Kept lean in registers: occupancy (many warps,
// each with a few KB in flight) is what saturates HBM on this random-block gather.
template <int G, int R, int PF, class PosT, bool DISTINCT, bool GEN>
__global__ void __launch_bounds__(kWarps * 32, FEA_GATHER_MIN_BLOCKS)
    k_gather_node(const double* __restrict__ K, const int64_t* __restrict__ adj_ptr,
             const int32_t* __restrict__ adj, const PosT* __restrict__ posA,
             const int64_t* __restrict__ nptr, const int32_t* __restrict__ order, int64_t n_own,
             int d, int npe, int pstride, int acc_stride, int pos_stride, int accumulate,
             int keep_k_in_l2, GenK gen, double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int GPW = 32 / G;
    const int m = d * npe;
    const int dm = d * m;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int gw = lane / G;
    const int warp = threadIdx.x >> 5;
    const int grp = warp * GPW + gw;
    double* acc = sacc + static_cast<int64_t>(grp) * acc_stride;
    PosT* spos = reinterpret_cast<PosT*>(sacc + static_cast<int64_t>(kWarps) * GPW * acc_stride) +
                 static_cast<int64_t>(grp) * pos_stride;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));

    // chunk-independent decode of this lane's entries, packed ki | b<<10 | kj<<20
    uint32_t tab[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int idx = r * G + gl;
        const int ki = idx / m;
        const int j = idx - ki * m;
        const int b = j / d;
        tab[r] = idx < dm ? (static_cast<uint32_t>(ki) | (static_cast<uint32_t>(b) << 10) |
                             (static_cast<uint32_t>(j - b * d) << 20))
                          : 0u;
    }

    const int64_t vi = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * GPW + gw;
    const int64_t v = (order != nullptr && vi < n_own) ? order[vi] : vi;
    int64_t b0 = 0, vb = 0;
    int n = 0, rowlen = 0, block = 0;
    if (vi < n_own) {
        b0 = adj_ptr[v];
        n = static_cast<int>(adj_ptr[v + 1] - b0);
        const int64_t c0 = nptr[v];
        rowlen = static_cast<int>(d * (nptr[v + 1] - c0));
        block = d * rowlen;
        vb = static_cast<int64_t>(d) * d * c0;
    }
    // the node's incidences (lane gl holds entry gl when n <= G) and position slice
    const int32_t my_ent = gl < n ? adj[b0 + gl] : 0;
    {
        const int np = n * npe;
        for (int q = gl; q < np; q += G) {
            const int k = q / npe;
            spos[q] = posA[(b0 + k) * pstride + (q - k * npe)];
        }
    }
    if (accumulate) {
        for (int i = gl; i < block; i += G) acc[i] = values[vb + i];
    } else {
        for (int i = gl; i < block; i += G) acc[i] = 0.0;
    }
    const int n_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));
    __syncwarp();

    double kv[PF][R];
    auto entry_of = [&](int k) -> int32_t {
        const int32_t e = __shfl_sync(0xffffffffu, my_ent, (gw * G + (k & (G - 1))) & 31);
        return n <= G ? e : (k < n ? adj[b0 + k] : 0);
    };
    auto load = [&](int p, int k) {
        const int32_t entry = entry_of(k);
        if (k < n) {
            if (GEN) {  // fused supplier
                const int64_t krow = entry / npe;
                const int a = static_cast<int>(entry - krow * npe);
                const uint64_t he = kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int idx = r * G + gl;
                    if (idx < dm) {
                        const uint32_t t = tab[r];
                        kv[p][r] = kgen_entry(he, a * d + static_cast<int>(t & 1023u),
                                              static_cast<int>((t >> 10) & 1023u) * d + static_cast<int>(t >> 20));
                    }
                }
            } else {
                const double* src = K + static_cast<int64_t>(entry) * dm;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int idx = r * G + gl;
                    // row blocks smaller than a 128 B line: keep lines in L2 for the element's
                    // other nodes (traversed close in time); else stream (read exactly once)
                    if (idx < dm) kv[p][r] = keep_k_in_l2 ? __ldcg(src + idx) : ld_stream(src + idx);
                }
            }
        }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) load(p, p);

    for (int k0 = 0; k0 < n_max; k0 += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int k = k0 + p;
            int q[R];
            if (k < n) {
                const PosT* pk = spos + k * npe;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t t = tab[r];
                    q[r] = static_cast<int>(t & 1023u) * rowlen +
                           static_cast<int>(pk[(t >> 10) & 1023u]) * d + static_cast<int>(t >> 20);
                    FEA_DCHECK(r * G + gl >= dm || (q[r] >= 0 && q[r] < block));
                }
            }
            if (DISTINCT) {
                // the slots of one element row block are distinct (no repeated node in an
                // element): all loads, then all adds, then all stores
                if (k < n) {
                    double a[R];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (r * G + gl < dm) a[r] = acc[q[r]];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (r * G + gl < dm) acc[q[r]] = a[r] + kv[p][r];
                }
            } else {
                // a repeated node: two entries of the row block share a slot; fold them one
                // entry at a time in entry order (idx = r*G + lane ascending = column order)
#pragma unroll
                for (int r = 0; r < R; ++r)
                    for (int l = 0; l < G; ++l) {
                        if (k < n && gl == l && r * G + gl < dm) acc[q[r]] += kv[p][r];
                        __syncwarp();
                    }
            }
            __syncwarp();
            load(p, k + PF);
        }
    }
    (void)gmask;
    for (int i = gl; i < block; i += G) __stcs(values + vb + i, acc[i]);
}

// ---------------------------------------------------------------------------
// Deterministic owner-computes gather, persistent streaming form (FEA_DET_SORTED)
// ---------------------------------------------------------------------------
// A group of G lanes owns a contiguous range of nodes [va, vb); each node's d rows
// are one contiguous block of values. Incidence lists of consecutive nodes are
// contiguous, so the group's work is ONE stream of element-matrix row blocks
// ("chunks") K[e][a*d..a*d+d-1][:], chunk t = adj[t] for t in
// [adj_ptr[va], adj_ptr[vb]), segmented by node — a CSR segmented reduction. The
// group keeps PF chunks in flight in registers (R rounds of G doubles each),
// continuously across node boundaries. Chunk indices and position-map words are
// staged through a per-group shared-memory ring: loaded into registers one block
// (kBlk chunks) early and stored when the block before is finished, so no
// dependent global load ever sits between two chunk loads. Each chunk is folded
// into the node's shared accumulator in ascending element order (group-local
// __syncwarp between chunks: a per-slot left fold from the slot's start value,
// bit-identical to assemble_sequential, assembly.hpp:112-118); at a node boundary
// the block is written once with coalesced streaming stores. K is read exactly
// once, values written once, no atomics.
constexpr int kPosW = 8;  // max position-map words staged per lane per block
template <int G>
constexpr int blk_of() { return G < 16 ? 16 : G; }  // chunks per staging block (>= G)

template <int R>
constexpr int gather_min_blocks() { return R >= 8 ? FEA_GATHER_MIN_BLOCKS_WIDE : FEA_GATHER_MIN_BLOCKS; }

template <int G, int R, int PF, class PosT, bool DISTINCT>
__global__ void __launch_bounds__(kWarps * 32, gather_min_blocks<R>())
    k_gather_stream(const double* __restrict__ K, const int64_t* __restrict__ adj_ptr,
             const int32_t* __restrict__ adj, const PosT* __restrict__ posA,
             const int64_t* __restrict__ nptr, int64_t n_own, int64_t n_groups, int d, int npe,
             int pstride, int acc_stride, int accumulate, double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int GPW = 32 / G;
    constexpr int kBlk = blk_of<G>();
    constexpr int EPL = kBlk / G;  // staged chunk indices per lane per block
    const int m = d * npe;
    const int dm = d * m;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int gw = lane / G;
    const int warp = threadIdx.x >> 5;
    const int grp = warp * GPW + gw;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
    const int pw_blk = kBlk * pstride * static_cast<int>(sizeof(PosT)) / 4;  // words per block
    double* acc = sacc + static_cast<int64_t>(grp) * acc_stride;
    int32_t* ring = reinterpret_cast<int32_t*>(sacc + static_cast<int64_t>(kWarps) * GPW * acc_stride) +
                    static_cast<int64_t>(grp) * 2 * (kBlk + pw_blk);
    int32_t* ent_ring = ring;                 // [2][kBlk]
    uint32_t* pos_ring = reinterpret_cast<uint32_t*>(ring + 2 * kBlk);  // [2][pw_blk] words

    uint32_t tab[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int idx = r * G + gl;
        const int ki = idx / m;
        const int j = idx - ki * m;
        const int b = j / d;
        tab[r] = idx < dm ? (static_cast<uint32_t>(ki) | (static_cast<uint32_t>(b) << 10) |
                             (static_cast<uint32_t>(j - b * d) << 20))
                          : 0u;
    }

    const int64_t g = (static_cast<int64_t>(blockIdx.x) * kWarps + warp) * GPW + gw;
    const int64_t va = n_own * g / n_groups;
    const int64_t vend = n_own * (g + 1) / n_groups;
    if (va >= vend) return;
    const int64_t t0 = adj_ptr[va];
    const int64_t t_end = adj_ptr[vend];
    const uint32_t* pos_words = reinterpret_cast<const uint32_t*>(posA);
    const int64_t pw_end = t_end * pstride * static_cast<int64_t>(sizeof(PosT)) / 4;

    int32_t se[EPL];
    uint32_t sp[kPosW];
    auto load_block = [&](int64_t blk) {
        const int64_t tb = t0 + blk * kBlk;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
            const int64_t t = tb + i * G + gl;
            se[i] = t < t_end ? adj[t] : 0;
        }
        const int64_t wb = tb * pstride * static_cast<int64_t>(sizeof(PosT)) / 4;
#pragma unroll
        for (int i = 0; i < kPosW; ++i) {
            const int q = i * G + gl;
            if (q < pw_blk && wb + q < pw_end) sp[i] = pos_words[wb + q];
        }
    };
    auto store_block = [&](int64_t blk) {
        const int slot = static_cast<int>(blk & 1);
#pragma unroll
        for (int i = 0; i < EPL; ++i) ent_ring[slot * kBlk + i * G + gl] = se[i];
#pragma unroll
        for (int i = 0; i < kPosW; ++i) {
            const int q = i * G + gl;
            if (q < pw_blk) pos_ring[slot * pw_blk + q] = sp[i];
        }
    };
    load_block(0);
    store_block(0);
    load_block(1);
    store_block(1);
    load_block(2);
    __syncwarp(gmask);

    int64_t v = va;
    int64_t seg_end = adj_ptr[v + 1];
    int64_t c0 = nptr[v];
    int rowlen = static_cast<int>(d * (nptr[v + 1] - c0));
    int block = d * rowlen;
    int64_t vbase = static_cast<int64_t>(d) * d * c0;
    for (int i = gl; i < block; i += G) acc[i] = accumulate ? values[vbase + i] : 0.0;
    __syncwarp(gmask);

    double kv[PF][R];
    auto issue = [&](int p, int64_t t) {
        if (t < t_end) {
            const int32_t e = ent_ring[(t - t0) & (2 * kBlk - 1)];
            const double* src = K + static_cast<int64_t>(e) * dm;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r * G + gl < dm) kv[p][r] = ld_stream(src + r * G + gl);
        }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) issue(p, t0 + p);

    const PosT* pos_ring_t = reinterpret_cast<const PosT*>(pos_ring);
    for (int64_t tt = t0; tt < t_end; tt += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int64_t t = tt + p;
            if (t < t_end) {
                while (t >= seg_end) {  // node boundary: write the finished block(s)
                    for (int i = gl; i < block; i += G) __stcs(values + vbase + i, acc[i]);
                    ++v;
                    seg_end = adj_ptr[v + 1];
                    c0 = nptr[v];
                    rowlen = static_cast<int>(d * (nptr[v + 1] - c0));
                    block = d * rowlen;
                    vbase = static_cast<int64_t>(d) * d * c0;
                    __syncwarp(gmask);
                    for (int i = gl; i < block; i += G) acc[i] = accumulate ? values[vbase + i] : 0.0;
                    __syncwarp(gmask);
                }
                const int64_t rel = t - t0;
                if ((rel & (kBlk - 1)) == 0 && rel > 0) {  // staging block boundary
                    const int64_t blk = rel / kBlk;
                    store_block(blk + 1);  // into the slot of block blk-1 (finished)
                    load_block(blk + 2);
                    __syncwarp(gmask);
                }
                const PosT* pk = pos_ring_t + (rel & (2 * kBlk - 1)) * pstride;
                int q[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t tb = tab[r];
                    q[r] = static_cast<int>(tb & 1023u) * rowlen +
                           static_cast<int>(pk[(tb >> 10) & 1023u]) * d + static_cast<int>(tb >> 20);
                    FEA_DCHECK(r * G + gl >= dm || (q[r] >= 0 && q[r] < block));
                }
                if (DISTINCT) {  // slots of one chunk are distinct: loads, adds, then stores
                    double a[R];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (r * G + gl < dm) a[r] = acc[q[r]];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (r * G + gl < dm) acc[q[r]] = a[r] + kv[p][r];
                } else {  // a repeated node: shared slots, folded entry by entry in entry order
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        for (int l = 0; l < G; ++l) {
                            if (gl == l && r * G + gl < dm) acc[q[r]] += kv[p][r];
                            __syncwarp(gmask);
                        }
                }
                __syncwarp(gmask);
                issue(p, t + PF);
            }
        }
    }
    for (;;) {  // the last node and any trailing empty nodes of the range
        for (int i = gl; i < block; i += G) __stcs(values + vbase + i, acc[i]);
        if (++v >= vend) break;
        c0 = nptr[v];
        rowlen = static_cast<int>(d * (nptr[v + 1] - c0));
        block = d * rowlen;
        vbase = static_cast<int64_t>(d) * d * c0;
        __syncwarp(gmask);
        for (int i = gl; i < block; i += G) acc[i] = accumulate ? values[vbase + i] : 0.0;
        __syncwarp(gmask);
    }
}

// ---------------------------------------------------------------------------
// Deterministic gather, lane = column node (FEA_DET_SORTED; G >= npe, D = d compile-time)
// ---------------------------------------------------------------------------
// The d x d sub-block K[e][a*d+ki][b*d+kj] of an incident row block lands in the d x d block
// of the node's values at column position pos(b): slot = ki*rowlen + pos(b)*d + kj. With lane
// = column node b and the D*D rounds = (ki, kj) unrolled at compile time, each lane does ONE
// position lookup per row block and every slot is a compile-time offset plus one add — the
// per-entry decode of k_gather_node disappears. The strided K loads (lane b reads d
// consecutive doubles of each of the d rows) go through L1 (ld.global.nc), which coalesces
// them back into whole sectors; DRAM traffic is unchanged. Fold order per slot as in
// k_gather_node: ascending element id, bit-identical to assemble_sequential.
#ifndef FEA_CN_MINB
#define FEA_CN_MINB 6
#endif
template <int G, int PF>
constexpr int cn_min_blocks() {  // warp-wide groups with one row block in flight fit 64 registers
#ifdef FEA_CN32_MINB
    return G == 32 ? FEA_CN32_MINB : FEA_CN_MINB;
#else
    return G == 32 && PF == 1 ? 8 : FEA_CN_MINB;
#endif
}
template <int G, int D, int PF, class PosT, bool DISTINCT, bool GEN>
__global__ void __launch_bounds__(kWarps * 32, cn_min_blocks<G, PF>())
    k_gather_cn(const double* __restrict__ K, const int64_t* __restrict__ adj_ptr,
                const int32_t* __restrict__ adj, const PosT* __restrict__ posA,
                const int64_t* __restrict__ nptr, const int32_t* __restrict__ order, int64_t n_own,
                int npe, int pstride, int acc_stride, int pos_stride, int accumulate, GenK gen,
                int64_t cta_acc, double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int GPW = 32 / G;
    constexpr int R = D * D;
    const int m = D * npe;
    const int dm = D * m;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int gw = lane / G;
    const int warp = threadIdx.x >> 5;
    const int grp = warp * GPW + gw;
    const bool col_ok = gl < npe;
    const int64_t vi = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * GPW + gw;
    const int64_t v = (order != nullptr && vi < n_own) ? order[vi] : vi;
    int64_t b0 = 0, vb = 0;
    int n = 0, rowlen = 0, block = 0;
    if (vi < n_own) {
        b0 = adj_ptr[v];
        n = static_cast<int>(adj_ptr[v + 1] - b0);
        const int64_t c0 = nptr[v];
        rowlen = static_cast<int>(D * (nptr[v + 1] - c0));
        block = D * rowlen;
        vb = static_cast<int64_t>(D) * D * c0;
    }
    // accumulators: acc_stride doubles per group, or (cta_acc > 0) packed — group g of the CTA
    // starts after the blocks (+1 bank stagger) of groups 0..g-1, cta_acc = the largest CTA total
    // (node rows differ in length, e.g. 125 / 75 / 45 / 27 column nodes on hex27)
    int64_t acc_off = static_cast<int64_t>(grp) * acc_stride;
    if (cta_acc > 0) {
        acc_off = 0;
        const int64_t vi0 = static_cast<int64_t>(blockIdx.x) * kWarps * GPW;
        for (int g = 0; g < grp; ++g) {
            if (vi0 + g >= n_own) break;
            const int64_t u = order != nullptr ? order[vi0 + g] : vi0 + g;
            acc_off += static_cast<int64_t>(D) * D * (nptr[u + 1] - nptr[u]) + 1;
        }
    }
    double* acc = sacc + acc_off;
    PosT* spos = reinterpret_cast<PosT*>(sacc + (cta_acc > 0 ? static_cast<int64_t>(cta_acc)
                                                              : static_cast<int64_t>(kWarps) * GPW * acc_stride)) +
                 static_cast<int64_t>(grp) * pos_stride;
    const int32_t my_ent = gl < n ? adj[b0 + gl] : 0;
    // the first row blocks' K loads depend only on the incidence list: issue them before
    // the position/accumulator set-up so their latency overlaps it
    double kv[PF][R];
    auto load = [&](int p, int k) {
        const int32_t e0 = __shfl_sync(0xffffffffu, my_ent, (gw * G + (k & (G - 1))) & 31);
        const int32_t entry = n <= G ? e0 : (k < n ? adj[b0 + k] : 0);
        if (k < n && col_ok) {
            if (GEN) {  // fused supplier: generate the d x d sub-block in registers
                const int64_t krow = entry / npe;
                const int a = static_cast<int>(entry - krow * npe);
                const uint64_t he = kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow);
#pragma unroll
                for (int ki = 0; ki < D; ++ki)
#pragma unroll
                    for (int kj = 0; kj < D; ++kj) kv[p][ki * D + kj] = kgen_entry(he, a * D + ki, gl * D + kj);
            } else {
                const double* src = K + static_cast<int64_t>(entry) * dm + gl * D;
#pragma unroll
                for (int ki = 0; ki < D; ++ki)
#pragma unroll
                    for (int kj = 0; kj < D; ++kj) kv[p][ki * D + kj] = __ldg(src + ki * m + kj);
            }
        }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) load(p, p);
    {   // the node's position rows, copied as 4-byte words in posA's layout (pstride per
        // incidence): all loads in flight before the stores (a byte-wise copy loop was a chain
        // of dependent load -> store round trips, 12 % of the stall samples on hex27)
        const uint32_t* src = reinterpret_cast<const uint32_t*>(posA + b0 * pstride);
        uint32_t* dst = reinterpret_cast<uint32_t*>(spos);
        const int words = n * pstride * static_cast<int>(sizeof(PosT)) / 4;
        constexpr int U = 4;
        for (int q0 = 0; q0 < words; q0 += U * G) {
            uint32_t w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + u * G + gl;
                w[u] = q < words ? src[q] : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + u * G + gl;
                if (q < words) dst[q] = w[u];
            }
        }
    }
    for (int i = gl; i < block; i += G) acc[i] = accumulate ? values[vb + i] : 0.0;
    const int n_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));
    __syncwarp();


    for (int k0 = 0; k0 < n_max; k0 += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int k = k0 + p;
            if (!DISTINCT) {
                // a repeated node: two lanes (columns) share slots; fold lane by lane in column order
                for (int l = 0; l < G; ++l) {
                    if (k < n && col_ok && gl == l) {
                        const int base = static_cast<int>(spos[k * pstride + gl]) * D;
#pragma unroll
                        for (int ki = 0; ki < D; ++ki)
#pragma unroll
                            for (int kj = 0; kj < D; ++kj) acc[ki * rowlen + base + kj] += kv[p][ki * D + kj];
                    }
                    __syncwarp();
                }
            } else if (k < n && col_ok) {
                const int base = static_cast<int>(spos[k * pstride + gl]) * D;
                FEA_DCHECK(base + (D - 1) * rowlen + D - 1 < block);
                {
                    double a[R];
#pragma unroll
                    for (int ki = 0; ki < D; ++ki)
#pragma unroll
                        for (int kj = 0; kj < D; ++kj) a[ki * D + kj] = acc[ki * rowlen + base + kj];
#pragma unroll
                    for (int ki = 0; ki < D; ++ki)
#pragma unroll
                        for (int kj = 0; kj < D; ++kj)
                            acc[ki * rowlen + base + kj] = a[ki * D + kj] + kv[p][ki * D + kj];
                }
            }
            __syncwarp();
            load(p, k + PF);
        }
    }
    for (int i = gl; i < block; i += G) __stcs(values + vb + i, acc[i]);
}

// Fixed-stride record form of k_gather_cn for warp-wide groups (G = 32: hex27, npe <= 28,
// <= 8 incidences per node, byte positions). k_gather_cn's node prologue is
// a chain of three memory round trips — adj_ptr / nptr, then the incidence entries and position
// rows at adj_ptr[v], then the K row blocks — and with ~3.3 incidences per hex27 node it is a
// third of the kernel's stall samples. Here a plan-time table holds, per traversal node at a
// fixed stride, a 16-byte header (values start, row length, incidence count, packed
// accumulator offset) and the node's incidence records {entry, position bytes} (8 x 32 B; one
// table per incidence order, so FEA_DET_COLOUR reads its colour-ordered records the same way):
// the warp loads both with one round trip (no adj_ptr dependence), then the K row blocks.
// Fold as k_gather_cn: ascending element id per slot, bit-identical.
constexpr int kCnrSlots = 8;   // incidence records per node
constexpr int kCnrBytes = 32;  // bytes per record: int32 entry + up to 28 position bytes
__global__ void k_cnr_build(const int32_t* __restrict__ order, const int64_t* __restrict__ adj_ptr,
                            const int32_t* __restrict__ adj, const uint8_t* __restrict__ posA,
                            const int64_t* __restrict__ nptr, int64_t n_own, int npe, int pstride, int d,
                            int per_cta, int4* __restrict__ hdr, int32_t* __restrict__ rec) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_own;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = order != nullptr ? order[t] : t;
        const int64_t b0 = adj_ptr[v];
        const int n = static_cast<int>(adj_ptr[v + 1] - b0);
        const int64_t c0 = nptr[v];
        const int cnt = static_cast<int>(nptr[v + 1] - c0);
        int64_t acc_off = 0;  // packed accumulators: blocks (+1 stagger) of the CTA's earlier groups
        for (int64_t g = t - t % per_cta; g < t; ++g) {
            const int64_t u = order != nullptr ? order[g] : g;
            acc_off += static_cast<int64_t>(d) * d * (nptr[u + 1] - nptr[u]) + 1;
        }
        const int64_t vb = static_cast<int64_t>(d) * d * c0;
        hdr[t] = make_int4(static_cast<int>(vb & 0xffffffff), static_cast<int>(vb >> 32),
                           d * cnt | (n << 16), static_cast<int>(acc_off));
        int32_t* r = rec + t * (kCnrSlots * kCnrBytes / 4);
        for (int k = 0; k < kCnrSlots; ++k) {
            uint32_t w[kCnrBytes / 4];
            for (int q = 0; q < kCnrBytes / 4; ++q) w[q] = 0;
            if (k < n) {
                w[0] = static_cast<uint32_t>(adj[b0 + k]);
                for (int b = 0; b < npe; ++b)
                    w[1 + b / 4] |= static_cast<uint32_t>(posA[(b0 + k) * pstride + b]) << (8 * (b & 3));
            }
            for (int q = 0; q < kCnrBytes / 4; ++q) r[k * (kCnrBytes / 4) + q] = static_cast<int32_t>(w[q]);
        }
    }
}

#ifndef FEA_CNR_MINB
#define FEA_CNR_MINB 6
#endif
#ifndef FEA_CNR_PF
#define FEA_CNR_PF 2
#endif
template <int D, int PF, bool GEN>
__global__ void __launch_bounds__(kWarps * 32, FEA_CNR_MINB)
    k_gather_cnr(const double* __restrict__ K, const int4* __restrict__ hdr, const int2* __restrict__ rec,
                 int64_t n_own, int npe, int accumulate, int64_t cta_acc, GenK gen, double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int R = D * D;
    const int m = D * npe;
    const int dm = D * m;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const bool col_ok = lane < npe;
    const int64_t vi = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    // one round trip: header and the node's 8 records (lane l: 8 bytes of the 256-byte block)
    int4 h = make_int4(0, 0, 0, 0);
    int2 rw = make_int2(0, 0);
    if (vi < n_own) {
        h = __ldg(hdr + vi);
        rw = __ldcs(rec + vi * 32 + lane);
    }
    int2* srec = reinterpret_cast<int2*>(sacc + cta_acc) + warp * 32;
    srec[lane] = rw;
    const int64_t vb = static_cast<int64_t>(static_cast<uint32_t>(h.x)) | (static_cast<int64_t>(h.y) << 32);
    const int rowlen = h.z & 0xffff;
    const int n = h.z >> 16;
    const int block = D * rowlen;
    double* acc = sacc + h.w;
    const uint8_t* spos = reinterpret_cast<const uint8_t*>(srec);
    const int32_t* sent = reinterpret_cast<const int32_t*>(srec);
    __syncwarp();
    double kv[PF][R];
    auto load = [&](int p, int k) {
        if (k < n && col_ok) {
            const int32_t entry = sent[k * (kCnrBytes / 4)];
            if (GEN) {  // fused supplier: generate the d x d sub-block in registers
                const int64_t krow = entry / npe;
                const int a = static_cast<int>(entry - krow * npe);
                const uint64_t he = kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow);
#pragma unroll
                for (int ki = 0; ki < D; ++ki)
#pragma unroll
                    for (int kj = 0; kj < D; ++kj) kv[p][ki * D + kj] = kgen_entry(he, a * D + ki, lane * D + kj);
            } else {
                const double* src = K + static_cast<int64_t>(entry) * dm + lane * D;
#pragma unroll
                for (int ki = 0; ki < D; ++ki)
#pragma unroll
                    for (int kj = 0; kj < D; ++kj) kv[p][ki * D + kj] = __ldg(src + ki * m + kj);
            }
        }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) load(p, p);
    for (int i = lane; i < block; i += 32) acc[i] = accumulate ? values[vb + i] : 0.0;
    __syncwarp();
    for (int k0 = 0; k0 < n; k0 += PF) {  // n is warp-uniform (one node per warp)
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int k = k0 + p;
            if (k < n && col_ok) {
                const int base = static_cast<int>(spos[k * kCnrBytes + 4 + lane]) * D;
                FEA_DCHECK(base + (D - 1) * rowlen + D - 1 < block);
                double a[R];
#pragma unroll
                for (int ki = 0; ki < D; ++ki)
#pragma unroll
                    for (int kj = 0; kj < D; ++kj) a[ki * D + kj] = acc[ki * rowlen + base + kj];
#pragma unroll
                for (int ki = 0; ki < D; ++ki)
#pragma unroll
                    for (int kj = 0; kj < D; ++kj) acc[ki * rowlen + base + kj] = a[ki * D + kj] + kv[p][ki * D + kj];
            }
            __syncwarp();
            load(p, k + PF);
        }
    }
    for (int i = lane; i < block; i += 32) __stcs(values + vb + i, acc[i]);
}

// ---------------------------------------------------------------------------
// Deterministic owner-computes gather for one DOF per node (d = 1): staged incidences
// ---------------------------------------------------------------------------
// With d = 1 a node's row block from one element is a single K row of npe doubles (32 B
// for tet4 / quad4): one sector per incidence and npe adds, so the per-node kernels above
// are bound by their prologue (order -> adj_ptr -> adj / posA: dependent global loads,
// then one dependent load per incidence) rather than by HBM. Here a group of G lanes
// (lane = column, G >= npe) owns one node: the prologue stages the node's incidence
// records {entry, position words} into shared memory with cp.async (all in flight at
// once), then the group folds them with PF K rows in flight; one shared load per step
// yields both the K address and the lane's slot. Groups of a CTA take consecutive
// traversal nodes (more nodes per group measured slower: the machine's working set then
// outgrows L2 reuse of the K lines the nodes share). Fold order per slot: ascending
// element id from the start value (assemble_sequential, assembly.hpp:112-118).
#ifndef FEA_D1_MINB
#define FEA_D1_MINB 12
#endif
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int G, int PF, class PosT, bool DISTINCT, bool GEN>
__global__ void __launch_bounds__(kWarps * 32, FEA_D1_MINB)
    k_gather_d1(const double* __restrict__ K, const int64_t* __restrict__ adj_ptr,
                const int32_t* __restrict__ adj, const PosT* __restrict__ posA,
                const int64_t* __restrict__ nptr, const int32_t* __restrict__ order, int64_t n_own,
                int npe, int pstride, int cap, int rec_stride, int acc_stride, int accumulate, int keep_k_in_l2,
                const int64_t* __restrict__ tptr, const int64_t* __restrict__ tmeta,
                const int32_t* __restrict__ trec, GenK gen, double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int gw = lane / G;
    const int grp = (threadIdx.x >> 5) * GPW + gw;
    const int pw = pstride * static_cast<int>(sizeof(PosT)) / 4;  // position words per incidence
    const int rw = pw == 1 ? 2 : (pw + 4) & ~3;                   // record words (int2 / int4 aligned)
    double* acc = sacc + static_cast<int64_t>(grp) * acc_stride;
    int32_t* rec = reinterpret_cast<int32_t*>(sacc + static_cast<int64_t>(kWarps) * GPW * acc_stride) +
                   static_cast<int64_t>(grp) * rec_stride;

    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarps * GPW + grp;
    int64_t a0 = 0, vb = 0;
    int n = 0, rl = 0;
    if (tptr != nullptr) {  // records pre-laid in traversal order: sequential reads
        if (t < n_own) {
            a0 = tptr[t];
            n = static_cast<int>(tptr[t + 1] - a0);
            const int64_t mt = tmeta[t];
            vb = mt >> 20;
            rl = static_cast<int>(mt & 0xfffff);
        }
        FEA_DCHECK(n <= cap);
        const int32_t* src = trec + a0 * rw;
        for (int i = gl; i < n * rw / 2; i += G) cp_async8(rec + 2 * i, src + 2 * i);
    } else {
        if (t < n_own) {
            const int64_t v = order != nullptr ? order[t] : t;
            a0 = adj_ptr[v];
            n = static_cast<int>(adj_ptr[v + 1] - a0);
            vb = nptr[v];
            rl = static_cast<int>(nptr[v + 1] - vb);
        }
        FEA_DCHECK(n <= cap);
        const uint32_t* pwords = reinterpret_cast<const uint32_t*>(posA + a0 * pstride);
        for (int i = gl; i < n; i += G) cp_async4(rec + i * rw, adj + a0 + i);
        for (int i = gl; i < n * pw; i += G) {
            const int k = i / pw;
            cp_async4(rec + k * rw + 1 + (i - k * pw), pwords + i);
        }
    }
    for (int i = gl; i < rl; i += G) acc[i] = accumulate ? values[vb + i] : 0.0;
    cp_async_wait_all();
    __syncwarp();
    const int n_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));

    const bool col_ok = gl < npe;
    // incidence k: element-matrix row (entry) and this lane's slot
    auto record = [&](int k, int32_t& entry) -> int {
        if (pw == 1) {
            const int2 r = *reinterpret_cast<const int2*>(rec + 2 * k);
            entry = r.x;
            constexpr int B = 8 * sizeof(PosT);
            return static_cast<int>((static_cast<uint32_t>(r.y) >> (B * gl)) & ((1u << B) - 1u));
        }
        entry = rec[k * rw];
        return static_cast<int>(reinterpret_cast<const PosT*>(rec + k * rw + 1)[gl]);
    };
    double kv[PF];
    int q[PF];
    auto load = [&](int p, int k) {
        if (k < n && col_ok) {
            int32_t entry;
            q[p] = record(k, entry);
            if (GEN) {
                const int64_t krow = entry / npe;
                const int a = static_cast<int>(entry - krow * npe);
                kv[p] = kgen_entry(kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow), a, gl);
            } else {
                const double* src = K + static_cast<int64_t>(entry) * npe + gl;
                kv[p] = keep_k_in_l2 ? __ldcg(src) : ld_stream(src);
            }
        }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) load(p, p);
    for (int k0 = 0; k0 < n_max; k0 += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int k = k0 + p;
            if (DISTINCT) {
                if (k < n && col_ok) {
                    FEA_DCHECK(q[p] < rl);
                    acc[q[p]] += kv[p];
                }
            } else {  // a repeated node: columns share a slot, folded lane by lane
                for (int l = 0; l < G; ++l) {
                    if (k < n && col_ok && gl == l) acc[q[p]] += kv[p];
                    __syncwarp();
                }
            }
            __syncwarp();
            load(p, k + PF);
        }
    }
    for (int i = gl; i < rl; i += G) __stcs(values + vb + i, acc[i]);
}

// Two-lane form of k_gather_d1 for the fused supplier (FEA_GEN: K generated in registers),
// npe = 4 (tet4 / quad4, d = 1) with traversal records: lane gl of a pair generates columns
// 2gl, 2gl+1 of the incidence's K row and folds both into the node's shared accumulator, so
// per warp instruction 16 nodes advance (8 in k_gather_d1) at half the instructions per entry
// (cfg3 fused: 0.89 -> 0.52 ms). With a materialized K this form measured slower (0.93 vs
// 0.64 ms: 9 CTAs/SM, shared-memory bound), so K loads use k_gather_d1g. Distinct element
// nodes only (a lane's two columns are distinct slots); per-slot fold order unchanged
// (ascending element id from the start value): same bits as k_gather_d1.
#ifndef FEA_D1V_MINB
#define FEA_D1V_MINB 10
#endif
template <int PF>
__global__ void __launch_bounds__(kWarps * 32, FEA_D1V_MINB)
    k_gather_d1v(int64_t n_own, int cap, int rec_stride, int acc_stride, int accumulate,
                 const int64_t* __restrict__ tptr,
                 const int64_t* __restrict__ tmeta, const int32_t* __restrict__ trec, GenK gen,
                 double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int G = 2;
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane & 1;
    const int grp = (threadIdx.x >> 1);
    double* acc = sacc + static_cast<int64_t>(grp) * acc_stride;
    int32_t* rec = reinterpret_cast<int32_t*>(sacc + static_cast<int64_t>(kWarps) * GPW * acc_stride) +
                   static_cast<int64_t>(grp) * rec_stride;

    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarps * GPW + grp;
    int64_t a0 = 0, vb = 0;
    int n = 0, rl = 0;
    if (t < n_own) {
        a0 = tptr[t];
        n = static_cast<int>(tptr[t + 1] - a0);
        const int64_t mt = tmeta[t];
        vb = mt >> 20;
        rl = static_cast<int>(mt & 0xfffff);
    }
    FEA_DCHECK(n <= cap);
    {
        const int32_t* src = trec + a0 * 2;
        for (int i = gl; i < n; i += G) cp_async8(rec + 2 * i, src + 2 * i);
    }
    for (int i = gl; i < rl; i += G) acc[i] = accumulate ? values[vb + i] : 0.0;
    cp_async_wait_all();
    __syncwarp();
    const int n_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));

    double2 kv[PF];
    uint32_t q[PF];  // the lane's two position bytes
    auto load = [&](int p, int k) {
        if (k < n) {
            const int2 r = *reinterpret_cast<const int2*>(rec + 2 * k);
            q[p] = static_cast<uint32_t>(r.y) >> (16 * gl);
            const int64_t krow = r.x >> 2;
            const int a = r.x & 3;
            const uint64_t he = kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow);
            kv[p].x = kgen_entry(he, a, 2 * gl);
            kv[p].y = kgen_entry(he, a, 2 * gl + 1);
        }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) load(p, p);
    for (int k0 = 0; k0 < n_max; k0 += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int k = k0 + p;
            if (k < n) {
                const int s0 = q[p] & 0xff, s1 = (q[p] >> 8) & 0xff;
                FEA_DCHECK(s0 < rl && s1 < rl);
                const double x0 = acc[s0], x1 = acc[s1];
                acc[s0] = x0 + kv[p].x;
                acc[s1] = x1 + kv[p].y;
            }
            __syncwarp();
            load(p, k + PF);
        }
    }
    for (int i = gl; i < rl; i += G) __stcs(values + vb + i, acc[i]);
}

// Direct-record form of k_gather_d1 (npe = 4, traversal records, materialized K): no record
// staging in shared memory (which capped residency at 12-13 CTAs/SM and cost a cp.async round
// trip per node); each lane reads the group's records straight from global memory through the
// read-only path (the 4 lanes of a group read the same 8 bytes; ld.global.nc, L1-cached: the
// streaming .cs form measured 0.60 vs 0.52 ms in tools/gather_probe_d1.py), U at a time, then
// the U K rows, then folds. Shared memory holds only the accumulators. Same fold order, bits.
#ifndef FEA_D1G_U
#define FEA_D1G_U 8  // records + K rows in flight per lane; cfg3: 4 -> 0.620 ms, 8 -> 0.614
#endif
#ifndef FEA_D1G_KLOAD
#define FEA_D1G_KLOAD 0  // K row loads: 0 L2 only (.cg), 1 read-only path (.nc, L1), 2 L1 (.ca)
#endif
__device__ __forceinline__ double kload_d1(const double* p) {
    if (FEA_D1G_KLOAD == 1) return __ldg(p);
    if (FEA_D1G_KLOAD == 2) return __ldca(p);
    return __ldcg(p);
}
#ifndef FEA_D1G_MINB
#define FEA_D1G_MINB 1
#endif
template <int U>
__global__ void __launch_bounds__(kWarps * 32, FEA_D1G_MINB)
    k_gather_d1g(const double* __restrict__ K, int64_t n_own, int acc_stride, int accumulate,
                 const int64_t* __restrict__ tptr, const int64_t* __restrict__ tmeta,
                 const int2* __restrict__ trec, double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int G = 4;
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane & 3;
    const int grp = threadIdx.x >> 2;
    double* acc = sacc + static_cast<int64_t>(grp) * acc_stride;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarps * GPW + grp;
    int64_t a0 = 0, vb = 0;
    int n = 0, rl = 0;
    if (t < n_own) {  // plan metadata: may run ahead of the previous kernel's end (PDL)
        a0 = tptr[t];
        n = static_cast<int>(tptr[t + 1] - a0);
        const int64_t mt = tmeta[t];
        vb = mt >> 20;
        rl = static_cast<int>(mt & 0xfffff);
    }
    const int n_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));
    const int2* src = trec + a0;
#ifndef FEA_D1G_PREFETCH
#define FEA_D1G_PREFETCH 0  // first record batch loaded before the PDL wait (+25 registers)
#endif
    int2 r0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r0[u] = FEA_D1G_PREFETCH && u < n ? __ldg(src + u) : make_int2(0, 0);
    pdl_wait();  // K and values only after the previous kernel of the stream has finished
    pdl_launch_dependents();
    for (int i = gl; i < rl; i += G) acc[i] = accumulate ? values[vb + i] : 0.0;
    for (int k0 = 0; k0 < n_max; k0 += U) {
        int2 r[U];
        double kv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            r[u] = (FEA_D1G_PREFETCH && k0 == 0) ? r0[u] : (k0 + u < n ? __ldg(src + k0 + u) : make_int2(0, 0));
#pragma unroll
        for (int u = 0; u < U; ++u)
            kv[u] = k0 + u < n ? kload_d1(K + static_cast<int64_t>(r[u].x) * 4 + gl) : 0.0;
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u < n) {
                const int q = (static_cast<uint32_t>(r[u].y) >> (8 * gl)) & 0xffu;
                FEA_DCHECK(q < rl);
                acc[q] += kv[u];
            }
            __syncwarp();
        }
    }
    for (int i = gl; i < rl; i += G) __stcs(values + vb + i, acc[i]);
}

// Lane-owned slots (npe = 4, d = 1, rows of <= 16 nodes, traversal records; materialized K).
// k_gather_d1g folds into a shared-memory accumulator at data-dependent slots: a bank-conflicted
// read-add-write per entry plus a warp barrier per incidence, and its 8-byte records cost 0.4 GB
// on cfg3. Here the plan has given every slot of the node's row to one lane of the node's
// group and one of that lane's accumulators (fea_plan::ln_*: lane 0 = the diagonal slot,
// lanes 1..3 = a 3-colouring of the node's link, so the 4 columns of every incident element
// fall on 4 distinct lanes), and every record tells lane c which column of the incidence's K
// row is its own and which accumulator it goes to: per incidence a lane does one 8-byte K load
// (the 4 lanes read the 4 doubles of one 32 B sector, as before) and one add into an
// accumulator no other lane touches - no warp synchronisation, no bank conflicts. Each slot
// still folds its contributions in record order from the start value: same bits.
// k_gather_d1s: 64 nodes per CTA, the lane's accumulators acc[q][thread] in shared memory, so
// the kernel fits 32 registers and 64 warps per SM. The bare access pattern (records -> K rows
// -> values, tools/gather_probe_d1.py) needs that residency: its dependent round trips per node
// are covered by nodes in flight, not by loads in flight per lane (U = 2..8, a record prefetch
// a batch ahead and every store cache policy measured within 2 %). Measured on cfg3 and
// dropped: register accumulators with one predicated add per register (66 registers, 28
// warps/SM: 0.626 ms; as plain C++ the compiler turns the register select into a jump table,
// 0.98 ms) and a persistent CTA whose node headers and records arrive by TMA bulk copies two
// tiles ahead with two K batches in flight per lane (56 registers: 0.92 ms, DRAM reads 2.67
// GB - the static tile stride lets CTAs drift apart and the K lines shared by neighbouring
// nodes leave L2), against 0.547 ms for this form with 8-byte records.
// Record word (LSB first): for lanes 1, 2, 3 in turn the element column the lane loads (2 bits)
// and its accumulator (wq1, wq2, wq3 bits, plan-wide widths), then - compact 4-byte records,
// used when it fits - the entry minus 4 * the node's lowest K row; 8-byte records keep the
// entry in a word of its own. Lane 0 owns only the node's diagonal slot: its column is
// entry & 3 (the bits right above the lane fields), its accumulator 0.
#ifndef FEA_D1S_U
#define FEA_D1S_U 4  // records + K rows in flight per lane (cfg3: 2, 4, 6, 8 within 2 %)
#endif
#ifndef FEA_D1S_MINB
#define FEA_D1S_MINB 8
#endif
constexpr int kD1sThreads = 256;
template <int U, bool REC4>
__global__ void __launch_bounds__(kD1sThreads, FEA_D1S_MINB)
    k_gather_d1s(const double* __restrict__ K, int64_t n_own, int accumulate, const int4* __restrict__ hdr,
                 const void* __restrict__ lrec, int q_max, int wq1, int wq2, int wq3,
                 double* __restrict__ values) {
    extern __shared__ double sacc[];
    constexpr int T = kD1sThreads;
    using Rec = typename std::conditional<REC4, uint32_t, int2>::type;
    const int gl = threadIdx.x & 3;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * (T / 4) + (threadIdx.x >> 2);
    int64_t vb = 0, a0 = 0;
    int n = 0, nq = 0;
    uint32_t lw = 0, base = 0;
    if (t < n_own) {  // plan metadata: may run ahead of the previous kernel's end (PDL)
        const int4 h0 = __ldg(hdr + 2 * t), h1 = __ldg(hdr + 2 * t + 1);
        const int64_t li = (static_cast<int64_t>(h0.y) << 32) | static_cast<uint32_t>(h0.x);
        const int64_t an = (static_cast<int64_t>(h0.w) << 32) | static_cast<uint32_t>(h0.z);
        vb = li >> 20;
        nq = static_cast<int>(li >> (4 * gl)) & 15;
        a0 = an & ((int64_t{1} << 40) - 1);
        n = static_cast<int>(an >> 40);
        base = static_cast<uint32_t>(h1.x);
        lw = gl == 0 ? (static_cast<uint32_t>(li >> 16) & 15u)
                     : static_cast<uint32_t>(gl == 1 ? h1.y : gl == 2 ? h1.z : h1.w);
    }
    const int n_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));
    const Rec* src = static_cast<const Rec*>(lrec) + a0;
    double* acc = sacc + threadIdx.x;
    // the lane's field of a record word: column at off, accumulator above it (mask mq)
    const int sh_e = 6 + wq1 + wq2 + wq3;
    const int off = gl == 0 ? sh_e : gl == 1 ? 0 : gl == 2 ? 2 + wq1 : 4 + wq1 + wq2;
    const uint32_t mq = gl == 0 ? 0u : (1u << (gl == 1 ? wq1 : gl == 2 ? wq2 : wq3)) - 1u;
    pdl_wait();  // K and values only after the previous kernel of the stream has finished
    pdl_launch_dependents();
    for (int q = 0; q < q_max; ++q)
        acc[q * T] = (accumulate && q < nq) ? values[vb + ((lw >> (4 * q)) & 15u)] : 0.0;
    for (int k0 = 0; k0 < n_max; k0 += U) {
        Rec r[U];
        double kv[U];
        int qv[U];
        // (ternaries, not branches: the loads stay predicated and issue back to back)
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = k0 + u < n ? __ldg(src + k0 + u) : Rec{};
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t w, ent;
            if constexpr (REC4) {
                w = r[u];
                ent = base + (w >> sh_e);
            } else {
                w = static_cast<uint32_t>(r[u].y);
                ent = static_cast<uint32_t>(r[u].x);
            }
            // lane 0: off points at the entry's low bits (8-byte records: taken from ent)
            const uint32_t f = (REC4 || gl != 0) ? w >> off : ent;
            kv[u] = k0 + u < n ? kload_d1(K + static_cast<int64_t>(ent) * 4 + (f & 3u)) : 0.0;
            qv[u] = static_cast<int>((f >> 2) & mq);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u < n) {
                FEA_DCHECK(qv[u] < nq);
                acc[qv[u] * T] += kv[u];
            }
    }
    for (int q = 0; q < q_max; ++q)
        if (q < nq) __stcs(values + vb + ((lw >> (4 * q)) & 15u), acc[q * T]);
}

// ---------------------------------------------------------------------------
// Deterministic owner-computes gather, lane = slot (d in {2,3,4}, npe <= 8, rows <= 32 nodes)
// ---------------------------------------------------------------------------
// The shared-memory accumulator of the kernels above costs a read-add-write per entry
// at data-dependent slots; on cfg2 those wavefronts (with bank conflicts) keep the L1 data
// pipe ~92 % busy. Here a WARP owns a node and lane s owns column node s of the node's row:
// its d x d values live in registers. The node's incident element row blocks ("chunks",
// d*m doubles each) are copied whole into shared memory with 16-byte cp.async (coalesced,
// no registers, all of a node's chunks in flight at once, double-buffered one node ahead);
// per chunk, lane s finds the element column that lands in its slot (byte compare on the
// position word) and adds that column's d x d sub-block from shared memory. Warps take
// nodes w, w + W, w + 2W, ... so the machine works on a contiguous window of nodes (the
// half lines two chunks of one element share stay in L2). Fold order per slot: ascending
// element id from the start value, then (repeated nodes) ascending column —
// assemble_sequential order (assembly.hpp:112-118), bit for bit.
#ifndef FEA_SLOT_TMA
#define FEA_SLOT_TMA 1
#endif
#ifndef FEA_SLOT_BRANCHLESS
#define FEA_SLOT_BRANCHLESS 1  // cfg2: 0.310 -> 0.278 ms (same bits)
#endif
#ifndef FEA_SLOT_WPC
// warps per CTA. Shared memory (9.5 KB per warp on cfg2 + 1 KB reserved per CTA) caps 4-warp
// CTAs at 5 per SM (20 warps); 8-warp CTAs fit 3 per SM (24 warps) but measured slower
// isolated (cfg2 0.307 vs 0.277 ms: the wider node window loses L2 reuse of shared half lines)
#define FEA_SLOT_WPC 4
#endif
constexpr int kSlotWarps = FEA_SLOT_WPC;
#ifndef FEA_SLOT_MINB
// register budget of 24 resident warps (swept with 4-warp CTAs: 4 (95 regs) 0.318 ms,
// 6 0.303, 8 0.305 on cfg2)
#define FEA_SLOT_MINB (24 / FEA_SLOT_WPC)
#endif
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__global__ void k_slot_fixed_build(const int32_t* __restrict__ order, const int64_t* __restrict__ adj_ptr,
                                   const int32_t* __restrict__ adj, const uint32_t* __restrict__ posw,
                                   const int64_t* __restrict__ nptr, int64_t n_own, int nbuf, int pw,
                                   int4* __restrict__ hdr, int4* __restrict__ rec) {
    const int lane = threadIdx.x & 31;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_own;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t v = order != nullptr ? order[t] : t;
        const int64_t a0 = adj_ptr[v];
        const int n = static_cast<int>(adj_ptr[v + 1] - a0);
        const int64_t c0 = nptr[v];
        if (lane == 0)
            hdr[t] = make_int4(static_cast<int>(c0 & 0xffffffff), static_cast<int>(c0 >> 32),
                               static_cast<int>(nptr[v + 1] - c0), n);
        for (int k = lane; k < nbuf; k += 32) {
            int4 r = make_int4(0, 0, 0, 0);
            if (k < n) {
                r.x = adj[a0 + k];
                r.y = static_cast<int>(posw[(a0 + k) * pw]);
                if (pw == 2) r.z = static_cast<int>(posw[(a0 + k) * pw + 1]);
            }
            rec[t * nbuf + k] = r;
        }
    }
}

// FIXED: per-node metadata from a plan-time table at a fixed stride — a 16-byte header
// {row start (int64), column count, incidence count} and nbuf 16-byte incidence records
// {entry, position words} — so a node's metadata is ONE round trip with no adj_ptr -> adj
// dependence (the same change took hex27's column-node gather 1.95 -> 1.78 ms).
template <int D, int NPE, bool DISTINCT, bool GEN, bool FIXED>
__global__ void __launch_bounds__(kSlotWarps * 32, FEA_SLOT_MINB)
    k_gather_slot(const double* __restrict__ K, const int64_t* __restrict__ adj_ptr,
                  const int32_t* __restrict__ adj, const uint8_t* __restrict__ posA,
                  const int64_t* __restrict__ nptr, const int32_t* __restrict__ order, int64_t n_own,
                  int nbuf, int istr, int accumulate, GenK gen, const int4* __restrict__ shdr,
                  const int4* __restrict__ srec, double* __restrict__ values) {
    extern __shared__ double sbuf[];
    constexpr int PW = NPE <= 4 ? 1 : 2;  // position words per incidence
    constexpr int npe = NPE;
    constexpr int m = D * NPE;
    constexpr int dm = D * m;     // doubles per chunk (even: 16-byte pieces)
    constexpr int half = dm / 2;  // 16-byte pieces per chunk
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    double* wbuf = sbuf + static_cast<int64_t>(warp) * 2 * nbuf * dm;
    const int64_t W = static_cast<int64_t>(gridDim.x) * kSlotWarps;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kSlotWarps + warp;

    // per-node pipeline: incidence range 3 nodes ahead, records (entry, position words) and
    // row info 2 ahead, chunk copies 1 ahead, fold of the current node
    struct Ptr {
        int64_t a0;
        int n;
    };
#if FEA_SLOT_BRANCHLESS
    // branch-free prefetch (clamped index, result masked): the loads' consumers are not pinned
    // right behind them by a branch join
    auto ptr_of = [&](int64_t t) -> Ptr {
        const bool ok = t < n_own;
        const int64_t tc = ok ? t : n_own - 1;
        const int64_t v = order != nullptr ? order[tc] : tc;
        Ptr P;
        P.a0 = adj_ptr[v];
        P.n = ok ? static_cast<int>(adj_ptr[v + 1] - P.a0) : 0;
        return P;
    };
#else
    auto ptr_of = [&](int64_t t) -> Ptr {
        Ptr P{0, 0};
        if (t < n_own) {
            const int64_t v = order != nullptr ? order[t] : t;
            P.a0 = adj_ptr[v];
            P.n = static_cast<int>(adj_ptr[v + 1] - P.a0);
        }
        return P;
    };
#endif
    struct Rec {
        int32_t ent;       // lane k: entry of incidence k
        uint32_t pw[PW];   // lane k: position words of incidence k
        int64_t c0;        // node row info (warp-uniform)
        int cnt, n;
    };
    auto rec_of = [&](const Ptr& P, int64_t t) -> Rec {
        Rec R;
        R.ent = 0;
#pragma unroll
        for (int w = 0; w < PW; ++w) R.pw[w] = 0;
        if constexpr (FIXED) {  // branch-free: clamped index, masked results
            const bool ok = t < n_own;
            const int64_t tc = ok ? t : n_own - 1;
            const int4 h = __ldg(shdr + tc);
            R.c0 = ok ? (static_cast<int64_t>(static_cast<uint32_t>(h.x)) | (static_cast<int64_t>(h.y) << 32)) : 0;
            R.cnt = ok ? h.z : 0;
            R.n = ok ? h.w : 0;
            if (lane < nbuf) {
                const int4 r = __ldg(srec + tc * nbuf + lane);
                R.ent = r.x;
                R.pw[0] = static_cast<uint32_t>(r.y);
                if (PW == 2) R.pw[PW - 1] = static_cast<uint32_t>(r.z);
            }
            return R;
        }
        R.n = P.n;
        R.c0 = 0;
        R.cnt = 0;
#if FEA_SLOT_BRANCHLESS
        {
            const bool ok = t < n_own;
            const int64_t tc = ok ? t : n_own - 1;
            const int64_t v = order != nullptr ? order[tc] : tc;
            const int64_t c0 = nptr[v];
            R.c0 = ok ? c0 : 0;
            R.cnt = ok ? static_cast<int>(nptr[v + 1] - c0) : 0;
        }
#else
        if (t < n_own) {
            const int64_t v = order != nullptr ? order[t] : t;
            R.c0 = nptr[v];
            R.cnt = static_cast<int>(nptr[v + 1] - R.c0);
        }
#endif
        if (lane < P.n) {
            R.ent = adj[P.a0 + lane];
            const uint32_t* src = reinterpret_cast<const uint32_t*>(posA) + (P.a0 + lane) * PW;
#pragma unroll
            for (int w = 0; w < PW; ++w) R.pw[w] = src[w];
        }
        return R;
    };
    // per-warp inverse position table: inv[k*istr + slot] = element column + 1 (0: none);
    // istr = the longest node row rounded to 4 bytes (<= 32)
    uint8_t* inv = reinterpret_cast<uint8_t*>(sbuf + static_cast<int64_t>(kSlotWarps) * 2 * nbuf * dm) +
                   static_cast<int64_t>(warp) * nbuf * istr;
#if FEA_SLOT_TMA
    // one mbarrier per buffer; lane k issues block k as ONE bulk copy (TMA), completion by bytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sbuf) +
                                                 static_cast<int64_t>(kSlotWarps) * nbuf * (2 * dm * 8 + istr)) +
                     2 * warp;
    if (!GEN && lane == 0) {
        mbar_init(smem_u32(bars), 1);
        mbar_init(smem_u32(bars + 1), 1);
        mbar_fence_init();
    }
    __syncwarp();
    uint32_t phase = 0;  // bit b: parity of buffer b's next completion
    auto issue = [&](const Rec& R, int b) {
        if (!GEN) {
            if (lane == 0) mbar_arrive_expect_tx(smem_u32(bars + b), static_cast<uint32_t>(R.n * dm * 8));
            __syncwarp();
            if (lane < R.n) {
                fence_proxy_async_smem();  // buffer b was last read by generic loads two nodes ago
                double* dst = wbuf + static_cast<int64_t>(b) * nbuf * dm + lane * dm;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(dst)),
                    "l"(K + static_cast<int64_t>(R.ent) * dm), "r"(dm * 8), "r"(smem_u32(bars + b))
                    : "memory");
            }
        }
    };
    auto wait_blocks = [&](int b) {
        if (!GEN) {
            mbar_wait(smem_u32(bars + b), (phase >> b) & 1u);
            phase ^= 1u << b;
        }
    };
#else
    auto issue = [&](const Rec& R, int b) {
        if (!GEN) {
            double* dst = wbuf + static_cast<int64_t>(b) * nbuf * dm;
            for (int k = 0; k < R.n; ++k) {  // chunk k: lanes copy its 16-byte pieces
                const int32_t e = __shfl_sync(0xffffffffu, R.ent, k);
                const double* src = K + static_cast<int64_t>(e) * dm;
#pragma unroll
                for (int pc = lane; pc < half; pc += 32) cp_async16(dst + k * dm + 2 * pc, src + 2 * pc);
            }
        }
        cp_async_commit();
    };
    auto wait_blocks = [&](int) { cp_async_wait_1(); };  // all but the newest group
#endif
    const uint32_t key = static_cast<uint32_t>(lane) * 0x01010101u;
    uint32_t valid[PW];
#pragma unroll
    for (int w = 0; w < PW; ++w) {
        const int nb = npe - 4 * w;
        valid[w] = nb >= 4 ? 0xffffffffu : nb <= 0 ? 0u : ((1u << (8 * nb)) - 1u);
    }

    const Ptr P0{0, 0};
    Rec Rc = rec_of(FIXED ? P0 : ptr_of(t0), t0);            // node j
    Rec R1 = rec_of(FIXED ? P0 : ptr_of(t0 + W), t0 + W);    // node j + 1
    Ptr P2 = FIXED ? P0 : ptr_of(t0 + 2 * W);                // node j + 2
    issue(Rc, 0);
    int b = 0;
    for (int64_t t = t0; t < n_own; t += W) {
        const Ptr P3 = FIXED ? P0 : ptr_of(t + 3 * W);
        const Rec R2 = rec_of(P2, t + 2 * W);
        issue(R1, b ^ 1);   // node j + 1's chunks, overlapping node j's fold
        wait_blocks(b);     // node j's chunks have landed
        __syncwarp();
        const double* cb = wbuf + static_cast<int64_t>(b) * nbuf * dm;
        const bool mine = lane < Rc.cnt;
        const int rowlen = D * Rc.cnt;
        double* vrow = values + static_cast<int64_t>(D) * D * Rc.c0 + lane * D;
        double acc[D][D];
#pragma unroll
        for (int ki = 0; ki < D; ++ki)
#pragma unroll
            for (int kj = 0; kj < D; ++kj) acc[ki][kj] = (accumulate && mine) ? vrow[ki * rowlen + kj] : 0.0;
        if constexpr (DISTINCT && !GEN) {
            // slots of one element are distinct: invert the position bytes once per node
            uint32_t* inv32 = reinterpret_cast<uint32_t*>(inv);
            for (int i = lane; i < Rc.n * (istr / 4); i += 32) inv32[i] = 0u;
            __syncwarp();
            for (int base = 0; base < Rc.n * NPE; base += 32) {  // warp-uniform trip count (shuffles)
                const int q = base + lane;
                const int k = q / NPE, col = q - k * NPE;
                // shuffle every word, then select: the source lane evaluates the shuffled operand
                const uint32_t w0 = __shfl_sync(0xffffffffu, Rc.pw[0], k & 31);
                const uint32_t w1 = PW == 1 ? w0 : __shfl_sync(0xffffffffu, Rc.pw[PW - 1], k & 31);
                const uint32_t w = col < 4 ? w0 : w1;
                if (q < Rc.n * NPE) inv[k * istr + ((w >> (8 * (col & 3))) & 0xffu)] = static_cast<uint8_t>(col + 1);
            }
            __syncwarp();
            if (mine) {
                for (int k = 0; k < Rc.n; ++k) {
                    const int c = inv[k * istr + lane];
                    if (c) {
                        const double* src = cb + k * dm + (c - 1) * D;
#pragma unroll
                        for (int ki = 0; ki < D; ++ki)
#pragma unroll
                            for (int kj = 0; kj < D; ++kj) acc[ki][kj] += src[ki * m + kj];
                    }
                }
            }
        } else
        for (int k = 0; k < Rc.n; ++k) {
            // bit 8*col set when element column node col lands in this lane's slot
            uint64_t mm = __vcmpeq4(__shfl_sync(0xffffffffu, Rc.pw[0], k), key) & valid[0] & 0x01010101u;
            if (PW == 2)
                mm |= static_cast<uint64_t>(__vcmpeq4(__shfl_sync(0xffffffffu, Rc.pw[PW - 1], k), key) &
                                            valid[PW - 1] & 0x01010101u) << 32;
            const int32_t e = GEN ? __shfl_sync(0xffffffffu, Rc.ent, k) : 0;
            if (!mine) continue;
            for (; mm; mm &= mm - 1) {  // DISTINCT: at most one column per slot
                const int col = (__ffsll(static_cast<long long>(mm)) - 1) >> 3;
                if (GEN) {
                    const int64_t krow = e / npe;
                    const int a = static_cast<int>(e - krow * npe);
                    const uint64_t he = kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow);
#pragma unroll
                    for (int ki = 0; ki < D; ++ki)
#pragma unroll
                        for (int kj = 0; kj < D; ++kj) acc[ki][kj] += kgen_entry(he, a * D + ki, col * D + kj);
                } else {
                    const double* src = cb + k * dm + col * D;
#pragma unroll
                    for (int ki = 0; ki < D; ++ki)
#pragma unroll
                        for (int kj = 0; kj < D; ++kj) acc[ki][kj] += src[ki * m + kj];
                }
                if (DISTINCT) break;
            }
        }
        if (mine) {
#pragma unroll
            for (int ki = 0; ki < D; ++ki)
#pragma unroll
                for (int kj = 0; kj < D; ++kj) __stcs(vrow + ki * rowlen + kj, acc[ki][kj]);
        }
        __syncwarp();  // buffer b is refilled two nodes on
        Rc = R1;
        R1 = R2;
        P2 = P3;
        b ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Element-owner scatter: atomics (FEA_ATOMIC) or plain adds within a colour
// ---------------------------------------------------------------------------
// tab[idx] = a | ki<<8 | b<<16 | kj<<24 for idx = i*m + j, i = a*d+ki, j = b*d+kj.
template <int G, class PosT, bool ATOMIC>
__global__ void __launch_bounds__(kWarps * 32)
    k_scatter(const double* __restrict__ K, const int32_t* __restrict__ list, int64_t n_list,
              const int32_t* __restrict__ elem_krow, const int32_t* __restrict__ conn_k,
              const PosT* __restrict__ posE, const int64_t* __restrict__ nptr, int64_t node_begin,
              int64_t n_own, int d, int npe, int serial, double* __restrict__ values) {
    extern __shared__ unsigned char smem[];
    constexpr int GPW = 32 / G;
    const int m = d * npe;
    const int mm = m * m;
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem);
    const int tab_words = (mm + 1) & ~1;
    int64_t* rb_all = reinterpret_cast<int64_t*>(tab + tab_words);
    int32_t* rl_all = reinterpret_cast<int32_t*>(rb_all + kWarps * GPW * npe);
    for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) {
        const int i = idx / m, j = idx - (idx / m) * m;
        const int a = i / d, b = j / d;
        tab[idx] = static_cast<uint32_t>(a) | (static_cast<uint32_t>(i - a * d) << 8) |
                   (static_cast<uint32_t>(b) << 16) | (static_cast<uint32_t>(j - b * d) << 24);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int gw = lane / G;
    const int warp = threadIdx.x >> 5;
    int64_t* rb = rb_all + (warp * GPW + gw) * npe;
    int32_t* rl = rl_all + (warp * GPW + gw) * npe;
    const int64_t stride_groups = ((int64_t)gridDim.x * blockDim.x >> 5) * GPW;
    for (int64_t gi = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * GPW + gw;
         gi - gw < n_list; gi += stride_groups) {
        const bool active = gi < n_list;
        int32_t le = 0, kr = 0;
        if (active) {
            le = list[gi];
            kr = elem_krow[le];
            for (int a = gl; a < npe; a += G) {
                const int64_t v = conn_k[static_cast<int64_t>(kr) * npe + a] - node_begin;
                const bool own = v >= 0 && v < n_own;
                rb[a] = own ? static_cast<int64_t>(d) * d * nptr[v] : -1;
                rl[a] = own ? static_cast<int32_t>(d * (nptr[v + 1] - nptr[v])) : 0;
            }
        }
        __syncwarp();
        if (active) {
            const double* src = K + static_cast<int64_t>(kr) * mm;
            const PosT* pe = posE + static_cast<int64_t>(le) * npe * npe;
            // a repeated node (serial): entries sharing a slot must be added in (i, j) order by
            // one lane (scatter_element, assembly.hpp:77-92); atomics need no order
            const int step = serial && !ATOMIC ? 1 : G;
#pragma unroll 4
            for (int idx = serial && !ATOMIC ? (gl == 0 ? 0 : mm) : gl; idx < mm; idx += step) {
                const uint32_t t = tab[idx];
                const int a = t & 0xff, ki = (t >> 8) & 0xff, b = (t >> 16) & 0xff, kj = t >> 24;
                const int64_t base = rb[a];
                const double x = ld_stream(src + idx);
                if (base >= 0) {
                    const int64_t s = base + static_cast<int64_t>(ki) * rl[a] +
                                      static_cast<int64_t>(pe[a * npe + b]) * d + kj;
                    FEA_DCHECK(s >= base && s < base + static_cast<int64_t>(d) * rl[a]);
                    if (ATOMIC) atomicAdd(values + s, x);
                    else values[s] += x;
                }
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Element-owner atomics, staged (FEA_ATOMIC for the common shapes)
// ---------------------------------------------------------------------------
// k_scatter above is bound by latency, not by the reductions: per element a chain of four
// dependent metadata loads (list -> elem_krow -> conn_k -> nptr), then one dependent position
// load per entry, with ~4 K loads in flight per lane (ncu: 75 % of stall samples on the REDs'
// operands, L2 36 % busy). Here the metadata is laid out in visit order at plan time
// (at_krow / at_rows / at_pos: sequential reads), and a warp streams a "step" of B elements
// (their K blocks, row words and position bytes) into shared memory with 16-byte cp.async,
// STAGES - 1 steps ahead, so the K bytes of several elements per warp are in flight while it
// issues the reductions of the current one. Entry -> slot: row word of the entry's row node
// (values start << 20 | row length, -1 off-partition) + ki * row length + pos * d + kj.
// One RED.E.ADD.F64 per entry, lanes on consecutive entries of the row-major block, as
// assemble_atomic (assembly.hpp:121-126) does one fetch_add per entry.
#ifndef FEA_AT_STAGES
#define FEA_AT_STAGES 3
#endif
#ifndef FEA_AT_MINB
#define FEA_AT_MINB 1
#endif
#ifndef FEA_AT_K_EVICT_FIRST
#define FEA_AT_K_EVICT_FIRST 1  // K is read once: keep the L2 for the values being reduced
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async16_hint(void* dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}
template <int D, int NPE, class PosT>
struct AtomicShape {
    static constexpr int M = D * NPE;
    static constexpr int MM = M * M;
    static constexpr int B = MM >= 128 ? 1 : 128 / MM;  // elements per warp step
    static constexpr int KD = B * MM;                    // K doubles per step
    static constexpr int T = (KD + 31) / 32;             // entries per lane per step
    static constexpr int RB = B * NPE * 8;               // row-word bytes per step
    static constexpr int PB = B * NPE * NPE * static_cast<int>(sizeof(PosT));  // position bytes per step
    static constexpr int STAGE = KD * 8 + RB + ((PB + 15) & ~15);
    static_assert(MM % 2 == 0 && RB % 16 == 0 && PB % 16 == 0, "16-byte staging pieces");
};

template <int D, int NPE, class PosT, int STAGES>
__global__ void __launch_bounds__(kWarps * 32, FEA_AT_MINB)
    k_atomic_staged(const double* __restrict__ K, const int32_t* __restrict__ at_krow,
                    const int64_t* __restrict__ at_rows, const PosT* __restrict__ at_pos, int64_t n_steps,
                    double* __restrict__ values) {
    using S = AtomicShape<D, NPE, PosT>;
    constexpr int M = S::M, MM = S::MM, B = S::B, KD = S::KD;
    extern __shared__ __align__(16) unsigned char smem_at[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    unsigned char* wbuf = smem_at + static_cast<size_t>(warp) * STAGES * S::STAGE;
    const int64_t W = static_cast<int64_t>(gridDim.x) * kWarps;
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    const uint64_t kpol = FEA_AT_K_EVICT_FIRST ? l2_policy_evict_first() : 0;

    // lane bb < B holds the K row of element bb of a step
    auto krow_of = [&](int64_t st) -> int32_t {
        return (st < n_steps && lane < B) ? at_krow[st * B + lane] : 0;
    };
    auto issue = [&](int stage, int64_t st, int32_t kr) {
        if (st < n_steps) {
            unsigned char* sb = wbuf + stage * S::STAGE;
            double* kd = reinterpret_cast<double*>(sb);
#pragma unroll
            for (int base = 0; base < KD / 2; base += 32) {  // warp-uniform trips (shuffles)
                const int pc = base + lane;
                const int bb = min(pc / (MM / 2), B - 1);
                const int32_t r = __shfl_sync(0xffffffffu, kr, bb);
                const double* src = K + static_cast<int64_t>(r) * MM + 2 * (pc - bb * (MM / 2));
                if (pc < KD / 2) {
                    if (FEA_AT_K_EVICT_FIRST) cp_async16_hint(kd + 2 * pc, src, kpol);
                    else cp_async16(kd + 2 * pc, src);
                }
            }
            const unsigned char* rs = reinterpret_cast<const unsigned char*>(at_rows + st * B * NPE);
            for (int pc = lane; pc < S::RB / 16; pc += 32) cp_async16(sb + KD * 8 + 16 * pc, rs + 16 * pc);
            const unsigned char* ps = reinterpret_cast<const unsigned char*>(at_pos) + st * S::PB;
            for (int pc = lane; pc < S::PB / 16; pc += 32) cp_async16(sb + KD * 8 + S::RB + 16 * pc, ps + 16 * pc);
        }
        cp_async_commit();
    };

    // prologue: STAGES - 1 steps in flight
    int32_t kr_next = 0;
#pragma unroll
    for (int k = 0; k < STAGES - 1; ++k) issue(k, s0 + k * W, krow_of(s0 + k * W));
    kr_next = krow_of(s0 + (STAGES - 1) * W);
    int stage = 0;
    for (int64_t st = s0; st < n_steps; st += W) {
        issue((stage + STAGES - 1) % STAGES, st + (STAGES - 1) * W, kr_next);
        kr_next = krow_of(st + STAGES * W);
        asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
        __syncwarp();
        const unsigned char* sb = wbuf + stage * S::STAGE;
        const double* kd = reinterpret_cast<const double*>(sb);
        const int64_t* rows = reinterpret_cast<const int64_t*>(sb + KD * 8);
        const PosT* pos = reinterpret_cast<const PosT*>(sb + KD * 8 + S::RB);
#pragma unroll
        for (int t = 0; t < S::T; ++t) {
            const int idx = lane + 32 * t;
            if (KD % 32 != 0 && idx >= KD) break;
            const int bb = idx / MM, r = idx - bb * MM;
            const int i = r / M, j = r - (r / M) * M;
            const int a = i / D, ki = i - a * D, b = j / D, kj = j - b * D;
            const int64_t w = rows[bb * NPE + a];
            if (w >= 0) {
                const int64_t slot = (w >> 20) + static_cast<int64_t>(ki) * (w & 0xfffff) +
                                     static_cast<int64_t>(pos[(bb * NPE + a) * NPE + b]) * D + kj;
                atomicAdd(values + slot, kd[idx]);
            }
        }
        __syncwarp();  // this stage is refilled by the next iteration's issue
        stage = (stage + 1) % STAGES;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// visit-order metadata for k_atomic_staged (padded to whole steps: row words -1, K row 0)
template <class PosT>
__global__ void k_atomic_maps(const int32_t* __restrict__ order, const int32_t* __restrict__ elem_krow,
                              const int32_t* __restrict__ conn_k, const int64_t* __restrict__ nptr,
                              const PosT* __restrict__ posE, int64_t E, int64_t E_pad, int npe, int d,
                              int64_t node_begin, int64_t n_own, int pstr, int32_t* __restrict__ at_krow,
                              int64_t* __restrict__ at_rows, PosT* __restrict__ at_pos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E_pad;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i >= E) {
            at_krow[i] = 0;
            for (int a = 0; a < npe; ++a) at_rows[i * npe + a] = -1;
            for (int q = 0; q < pstr; ++q) at_pos[i * pstr + q] = 0;
            continue;
        }
        const int32_t le = order[i];
        const int32_t kr = elem_krow[le];
        at_krow[i] = kr;
        for (int a = 0; a < npe; ++a) {
            const int64_t v = conn_k[static_cast<int64_t>(kr) * npe + a] - node_begin;
            int64_t w = -1;
            if (v >= 0 && v < n_own) {
                const int64_t c0 = nptr[v];
                w = ((static_cast<int64_t>(d) * d * c0) << 20) | (static_cast<int64_t>(d) * (nptr[v + 1] - c0));
            }
            at_rows[i * npe + a] = w;
        }
        for (int q = 0; q < pstr; ++q)
            at_pos[i * pstr + q] = q < npe * npe ? posE[static_cast<int64_t>(le) * npe * npe + q] : PosT(0);
    }
}

// ---------------------------------------------------------------------------
// Atomic route with patch pre-reduction (hex8-type shapes: npe = 8, d <= 3)
// ---------------------------------------------------------------------------
// k_atomic_staged issues one RED per element-matrix entry: cfg2's 151 M lanes become 64.6 M
// L2 reduction sectors, and that sector rate (~115e9/s), not HBM, bounds the route. Elements
// that share nodes add into the same d x d node-pair blocks, so the plan groups the elements
// into patches of up to P = 8 node-sharing elements (greedy growth by shared nodes from the
// visit order: 2 x 2 x 2 blocks on structured meshes, 343 distinct node pairs for 512 element
// node pairs) and lists each patch's distinct (row node, column node) pairs sorted by (row,
// position). A CTA owns a patch: it streams the patch's element blocks through shared memory
// (cp.async, STAGES - 1 elements ahead), adds every entry into the patch accumulator
// acc[pair][ki][kj] in shared memory (one element at a time, CTA barrier between elements:
// within an element the (a, b) node pairs are distinct, so threads never collide), then
// flushes it row by row — a warp per patch row, lanes over (ki, pair, kj), so the REDs of one
// warp instruction cover the row's consecutive pairs at consecutive addresses — with one RED
// per distinct slot. Conflicts between patches are still resolved by atomics only: this IS
// the atomic route (assemble_atomic, assembly.hpp:121-126), with fewer and denser reductions.
// Values match assemble_sequential within the reference tolerance (the pre-reduction changes
// the summation order like any atomic schedule does).
#ifndef FEA_PATCH_K_HINT
// K copies with an L2 evict-first policy: ptxas 12.9 folded the createpolicy of the first form
// of this kernel into uniform registers and then encoded the copies with unset descriptor
// registers (the launch died with "illegal instruction"); plain cp.async by default
#define FEA_PATCH_K_HINT 0
#endif
#ifndef FEA_PATCH_WARPS
#define FEA_PATCH_WARPS 4
#endif
constexpr int kPatchElems = 8;  // elements per patch (a 2 x 2 x 2 block of hex8)
constexpr int kPatchWarps = FEA_PATCH_WARPS;
template <int D, int NPE, int P, int STAGES>
__global__ void __launch_bounds__(kPatchWarps * 32)
    k_atomic_patch(const double* __restrict__ K, const int4* __restrict__ hdr, const int32_t* __restrict__ pk_krow,
                   const uint16_t* __restrict__ pk_cidx, const int64_t* __restrict__ pk_rows,
                   const int32_t* __restrict__ pk_rowpair, const uint16_t* __restrict__ pk_pairs, int64_t n_patch,
                   int acc_doubles, unsigned long long* __restrict__ ticket, double* __restrict__ values) {
    constexpr int M = D * NPE, MM = M * M, DD = D * D, NN = NPE * NPE;
    constexpr int KB = MM * 8, CB = NN * 2, SLOT = KB + CB;
    constexpr int NT = kPatchWarps * 32;
    constexpr int T = (MM + NT - 1) / NT;  // entries per thread per element
    static_assert(KB % 16 == 0 && CB % 16 == 0, "16-byte bulk copies");
    extern __shared__ __align__(16) unsigned char smem_pa[];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    double* acc = reinterpret_cast<double*>(smem_pa);
    unsigned char* stg = smem_pa + static_cast<size_t>(acc_doubles) * 8;
    // the patch's flush tables, staged once per patch (loaded into registers early in the
    // patch, stored before the flush): rows (values start | length), row pair ranges, pairs
    constexpr int MAXR = P * NPE, MAXP = P * NN;
    constexpr int PPT = (MAXP + NT - 1) / NT;
    int64_t* s_rows = reinterpret_cast<int64_t*>(stg + STAGES * SLOT);
    int32_t* s_rowpair = reinterpret_cast<int32_t*>(s_rows + MAXR);
    uint16_t* s_pairs = reinterpret_cast<uint16_t*>(s_rowpair + MAXR);
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_pairs + MAXP);  // one mbarrier per stage
    // patches are handed out in order by a ticket counter (zeroed by the launcher): persistent
    // CTAs striding by gridDim drift apart over thousands of patches, and the values rows that
    // neighbouring patches share (the next row of patches, 128 patches later on config 5) have
    // left L2 by the time the slower CTA reaches them. The issue cursor claims a patch, the
    // fold cursor picks it up from s_q a few slots later. ticket == nullptr: static stride (A/B).
    int64_t* s_q = reinterpret_cast<int64_t*>(bars + STAGES);  // 4 patch ids, issue -> fold cursor
    int64_t m_row = 0;
    int32_t m_rowpair = 0;
    uint16_t m_pair[PPT];
    const int64_t G = gridDim.x;
    int qw = 0, qr = 0;
    // thread 0 holds the ticket of the patch after the one its issue cursor is in, so the
    // counter's round trip (~1 us, 10 % of a patch on cfg2) is off the issue path
    auto ticket_next = [&](int64_t stride_next) -> int64_t {
        return ticket ? static_cast<int64_t>(atomicAdd(ticket, 1ull)) : stride_next;
    };
    int64_t ipt = 0, ipt_next = 0;
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) mbar_init(smem_u32(bars + st), 1);
        mbar_fence_init();
        ipt = ticket_next(blockIdx.x);
        ipt_next = ticket_next(ipt + G);
        s_q[qw++ & 3] = ipt;
    }
    __syncthreads();
    int64_t pt = s_q[qr++ & 3];
    if (pt >= n_patch) return;
    // K is read once: L2 evict-first for its bulk copies keeps the values lines being reduced
    // into resident (created per copy: a hoisted createpolicy was miscompiled, see above)
    // issue cursor (STAGES - 1 element slots ahead of the fold): patch and slot. Thread 0
    // copies a slot's K block (4.6 KB contiguous) and its pair indices with two bulk copies.
    int ik = 0;
    auto advance = [&]() {
        if (++ik == P) {
            ik = 0;
            ipt = ipt_next;
            s_q[qw++ & 3] = ipt;
            ipt_next = ticket_next(ipt + G);
        }
    };
    auto krow_at = [&]() -> int32_t { return ipt < n_patch ? __ldg(pk_krow + ipt * P + ik) : -1; };
    auto issue = [&](int stage, int32_t kr) {  // the slot at the cursor (thread 0 only)
        const uint32_t bar = smem_u32(bars + stage);
        if (kr >= 0) {
            unsigned char* sb = stg + stage * SLOT;
            fence_proxy_async_smem();  // the stage was last read by generic loads
            mbar_arrive_expect_tx(bar, SLOT);
            if (FEA_PATCH_K_HINT)
                tma_load_1d(smem_u32(sb), K + static_cast<int64_t>(kr) * MM, KB, bar, policy_evict_first());
            else bulk_g2s(smem_u32(sb), K + static_cast<int64_t>(kr) * MM, KB, bar);
            bulk_g2s(smem_u32(sb + KB), pk_cidx + (ipt * P + ik) * NN, CB, bar);
        } else {
            mbar_arrive(bar);  // empty slot: complete the phase without data
        }
    };
    // this thread's entries of an element block, decoded once into byte offsets: the entry's
    // pair-index slot in the staged indices and its (ki, kj) offset inside a pair's block
    uint32_t cio[T], co8[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int idx = min(tid + NT * t, MM - 1);
        const int i = idx / M, jj = idx - (idx / M) * M;
        cio[t] = static_cast<uint32_t>(((i / D) * NPE + jj / D) * 2);
        co8[t] = static_cast<uint32_t>(((i % D) * D + jj % D) * 8);
        // passed through a shuffle so the code generator keeps them in registers instead of
        // re-deriving them (two magic-number divisions and a dozen integer ops) for every entry
        // of every element (an empty asm does not stop ptxas from rematerializing)
        cio[t] = __shfl_sync(0xffffffffu, cio[t], lane);
        co8[t] = __shfl_sync(0xffffffffu, co8[t], lane);
    }
    constexpr int FQ = 32 / D;  // flush: lane = (pair in a chunk of FQ, kj), ki looped
    const int fq = lane / D, fkj = lane - (lane / D) * D;
    int32_t kr_next = -1;
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < STAGES - 1; ++k) {
            issue(k, krow_at());
            advance();
        }
        kr_next = krow_at();
    }
    int4 h = make_int4(0, 0, 0, 0);
    int k = 0, stage = 0;
    uint32_t phase = 0;  // bit st: parity of stage st's next completion
    for (; pt < n_patch;) {
        if (k == 0) {  // patch start: header, zero the accumulator (the barrier below orders it)
            h = __ldg(hdr + pt);
            const int n_pairs = static_cast<int>(static_cast<uint32_t>(h.w) >> 16);
            for (int f = tid; f < (n_pairs + 1) * DD; f += NT) acc[f] = 0.0;  // + the spare pair
        }
        mbar_wait(smem_u32(bars + stage), (phase >> stage) & 1u);
        phase ^= 1u << stage;
        __syncthreads();  // the previous slot's adds are done (acc ordering, stage reuse)
        if (tid == 0) {
            issue((stage + STAGES - 1) % STAGES, kr_next);
            advance();
            kr_next = krow_at();
        }
        if (k == (P > 1 ? 1 : 0)) {  // this patch's flush tables: loads in flight during the adds
            const int n_rows = (h.w >> 8) & 0xff, n_pairs = static_cast<int>(static_cast<uint32_t>(h.w) >> 16);
            if (tid < n_rows) {
                m_row = __ldg(pk_rows + h.z + tid);
                m_rowpair = __ldg(pk_rowpair + h.z + tid);
            }
#pragma unroll
            for (int u = 0; u < PPT; ++u)
                m_pair[u] = tid + NT * u < n_pairs ? __ldg(pk_pairs + h.y + tid + NT * u) : uint16_t(0);
        }
        if (k < (h.w & 0xff)) {
            // entries whose row node is not owned carry the spare pair index (never flushed)
            const unsigned char* sb = stg + stage * SLOT;
            const unsigned char* kb = sb + tid * 8;
            const unsigned char* cb = sb + KB;
            unsigned char* ab = reinterpret_cast<unsigned char*>(acc);
            // within one element the (a, b) pairs are distinct, so a thread's T entries land in T
            // different accumulator slots (or in the spare pair, never flushed): all index and K
            // loads first, then the accumulator loads, then the stores - one shared-memory round
            // trip per phase instead of a load -> add -> store chain per entry (ncu, config 5:
            // 30 % of the stall samples on those chains, 20 % on the barrier that waits for them)
            double kv[T], av[T];
            double* ap[T];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const bool on = t < T - 1 || MM % NT == 0 || tid + NT * t < MM;
                const uint32_t c = on ? *reinterpret_cast<const uint16_t*>(cb + cio[t]) : 0u;
                kv[t] = on ? *reinterpret_cast<const double*>(kb + t * NT * 8) : 0.0;
                ap[t] = reinterpret_cast<double*>(ab + c * (DD * 8) + co8[t]);
            }
#pragma unroll
            for (int t = 0; t < T; ++t) av[t] = *ap[t];
#pragma unroll
            for (int t = 0; t < T; ++t)
                if (t < T - 1 || MM % NT == 0 || tid + NT * t < MM) *ap[t] = av[t] + kv[t];
        }
        if (k == P - 1) {  // patch end: a warp per row, one RED per distinct slot
            const int n_rows = (h.w >> 8) & 0xff;
            if (tid < n_rows) {
                s_rows[tid] = m_row;
                s_rowpair[tid] = m_rowpair;
            }
#pragma unroll
            for (int u = 0; u < PPT; ++u) s_pairs[tid + NT * u] = m_pair[u];
            __syncthreads();
            for (int r = warp; r < n_rows; r += kPatchWarps) {
                const int64_t w = s_rows[r];
                const int32_t rp = s_rowpair[r];  // first pair | count << 16
                const int q0 = rp & 0xffff, cnt = rp >> 16;
                const int64_t rowlen = w & 0xfffff;
                double* vrow = values + (w >> 20) + fkj;
                for (int qb = 0; qb < cnt; qb += FQ) {
                    const int ql = qb + fq;
                    if (fq < FQ && ql < cnt) {
                        const int q = q0 + ql;
                        double* dst = vrow + (s_pairs[q] & 0xff) * D;
                        const double* src = acc + q * DD + fkj;
#pragma unroll
                        for (int ki = 0; ki < D; ++ki) atomicAdd(dst + ki * rowlen, src[ki * D]);
                    }
                }
            }
            __syncthreads();  // the accumulator is zeroed and the tables restaged for the next patch
        }
        stage = (stage + 1) % STAGES;
        if (++k == P) {
            k = 0;
            pt = s_q[qr++ & 3];  // claimed STAGES - 1 slots (and several barriers) ago
        }
    }
}

// Large element blocks (hex27: m = 81, a 52 KB block per element): one CTA per element step.
// The CTA stages only the step's row words and position bytes (double-buffered, cp.async);
// each thread loads ALL its entries of the block straight into registers (consecutive
// threads, consecutive doubles: coalesced; 26 loads in flight per thread) and reduces them.
// Staging the whole 52 KB block in shared memory instead (2 CTAs/SM) measured 3.48 ms on
// cfg4 vs 3.14 ms for this form (13 loads in flight per thread: 3.49 ms).
constexpr int kAtCtaThreads = 256;
template <int D, int NPE, class PosT>
struct AtomicCtaShape {
    static constexpr int M = D * NPE;
    static constexpr int MM = M * M;
    static constexpr int RB = (NPE * 8 + 15) & ~15;                                    // row words
    static constexpr int PSTR = (NPE * NPE * static_cast<int>(sizeof(PosT)) + 15) & ~15;  // position bytes
    static constexpr int STAGE = RB + PSTR + ((MM * 8 + 15) & ~15);
    static constexpr int T = (MM + kAtCtaThreads - 1) / kAtCtaThreads;
};

#ifndef FEA_AT_DIRECT_U
#define FEA_AT_DIRECT_U 26
#endif
#ifndef FEA_AT_DIRECT_MINB
#define FEA_AT_DIRECT_MINB 1
#endif
template <int D, int NPE, class PosT>
__global__ void __launch_bounds__(kAtCtaThreads, FEA_AT_DIRECT_MINB)
    k_atomic_direct(const double* __restrict__ K, const int32_t* __restrict__ at_krow,
                    const int64_t* __restrict__ at_rows, const PosT* __restrict__ at_pos, int64_t n_steps,
                    double* __restrict__ values) {
    using S = AtomicCtaShape<D, NPE, PosT>;
    constexpr int M = S::M, MM = S::MM, U = FEA_AT_DIRECT_U;
    constexpr int MST = S::RB + S::PSTR;  // metadata stage bytes
    __shared__ __align__(16) unsigned char smeta[2 * MST];
    const int tid = threadIdx.x;
    auto issue = [&](int stage, int64_t st) {
        if (st < n_steps) {
            unsigned char* sb = smeta + stage * MST;
            if (tid < NPE) cp_async8(sb + 8 * tid, at_rows + st * NPE + tid);
            const unsigned char* ps = reinterpret_cast<const unsigned char*>(at_pos) + st * S::PSTR;
            for (int q = tid; q < S::PSTR / 16; q += kAtCtaThreads) cp_async16(sb + S::RB + 16 * q, ps + 16 * q);
        }
        cp_async_commit();
    };
    int stage = 0;
    issue(0, blockIdx.x);
    int32_t kr_next = blockIdx.x < n_steps ? at_krow[blockIdx.x] : 0;
    for (int64_t st = blockIdx.x; st < n_steps; st += gridDim.x) {
        const int32_t kr = kr_next;
        issue(stage ^ 1, st + gridDim.x);
        kr_next = st + gridDim.x < n_steps ? at_krow[st + gridDim.x] : 0;
        cp_async_wait_1();
        __syncthreads();
        const unsigned char* sb = smeta + stage * MST;
        const int64_t* rows = reinterpret_cast<const int64_t*>(sb);
        const PosT* pos = reinterpret_cast<const PosT*>(sb + S::RB);
        const double* src = K + static_cast<int64_t>(kr) * MM;
        for (int t0 = 0; t0 < S::T; t0 += U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = tid + kAtCtaThreads * (t0 + u);
                v[u] = (t0 + u < S::T && idx < MM) ? ld_stream(src + idx) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = tid + kAtCtaThreads * (t0 + u);
                if (t0 + u < S::T && idx < MM) {
                    const int i = idx / M, j = idx - (idx / M) * M;
                    const int a = i / D, ki = i - a * D, b = j / D, kj = j - b * D;
                    const int64_t w = rows[a];
                    if (w >= 0) {
                        const int64_t slot = (w >> 20) + static_cast<int64_t>(ki) * (w & 0xfffff) +
                                             static_cast<int64_t>(pos[a * NPE + b]) * D + kj;
                        atomicAdd(values + slot, v[u]);
                    }
                }
            }
        }
        __syncthreads();
        stage ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Element-order maps for the element-owner routes (built lazily)
// ---------------------------------------------------------------------------
template <class PosT>
__global__ void k_pos_elem(const int32_t* __restrict__ adj, const PosT* __restrict__ posA,
                           int64_t n_adj, int npe, int pstride, const int32_t* __restrict__ k2l,
                           PosT* __restrict__ posE) {
    const int64_t total = n_adj * npe;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / npe;
        const int b = static_cast<int>(t - k * npe);
        const int32_t entry = adj[k];
        const int32_t kr = entry / npe;
        const int a = entry - kr * npe;
        const int64_t le = k2l ? k2l[kr] : kr;
        posE[(le * npe + a) * npe + b] = posA[k * pstride + b];
    }
}

__global__ void k_k2l(const int32_t* __restrict__ elem_krow, int64_t E, int32_t* __restrict__ k2l) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x)
        k2l[elem_krow[i]] = static_cast<int32_t>(i);
}

// consecutive-element node sharing (locality test) and min-node sort keys
__global__ void k_locality(const int32_t* __restrict__ conn_k, const int32_t* __restrict__ elem_krow,
                           int64_t E, int npe, unsigned long long* shared_pairs,
                           uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* c = conn_k + static_cast<int64_t>(elem_krow[i]) * npe;
        uint32_t mn = 0xffffffffu;
        for (int a = 0; a < npe; ++a) mn = min(mn, static_cast<uint32_t>(c[a]));
        keys[i] = mn;
        vals[i] = static_cast<int32_t>(i);
        if (i > 0) {
            const int32_t* q = conn_k + static_cast<int64_t>(elem_krow[i - 1]) * npe;
            bool sh = false;
            for (int a = 0; a < npe && !sh; ++a)
                for (int b = 0; b < npe; ++b)
                    if (c[a] == q[b]) { sh = true; break; }
            if (sh) atomicAdd(shared_pairs, 1ull);
        }
    }
}

__global__ void k_iota32(int32_t* x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = static_cast<int32_t>(i);
}

__global__ void k_fill_k(double* __restrict__ K, int64_t n, int m, uint64_t seed,
                         const int64_t* __restrict__ ids) {
    const int64_t mm = static_cast<int64_t>(m) * m;
    const int64_t total = n * mm;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t / mm;
        const int rem = static_cast<int>(t - e * mm);
        const int i = rem / m, j = rem - (rem / m) * m;
        K[t] = kval(seed, ids ? ids[e] : e, i, j);
    }
}

// ---------------------------------------------------------------------------
// FEA_ATOMIC for npe = 4, d = 1 (tet4 / quad4 scalar problems): strip pre-reduction
// ---------------------------------------------------------------------------
// Every atomic kernel here runs at the L2's fp64 atomic-add rate (~230e9 doubles/s, DESIGN.md
// §5), so this shape (16 entries per element, 201 M on cfg3) has to reduce fewer doubles. A CTA
// takes a strip of kStripElems consecutive elements of the visit order: one bulk copy brings
// the strip's K rows (6 KB, contiguous when the K rows are consecutive; else a 128-byte copy per
// element), one its record and one its shape (fea_plan::sk_meta / sk_shape: the shape table is
// de-duplicated and L2-resident on regular meshes). Thread t owns the t-th distinct slot of
// the strip: it sums the K entries that feed it from shared memory, in ascending entry order,
// and issues ONE reduction - no shared accumulators, no barrier between elements. On a Kuhn
// mesh a strip of 8 cubes has ~270 distinct slots for its 768 entries. Strips are handed out by
// ticket like the hex8 patches. Conflict resolution = assemble_atomic's (atomics between strips).
constexpr int kStripElems = 48;
constexpr int kStripThreads = 256;
#ifndef FEA_STRIP_STAGES
#define FEA_STRIP_STAGES 3
#endif
template <int STAGES>
__global__ void __launch_bounds__(kStripThreads)
    k_atomic_strip(const double* __restrict__ K, const unsigned char* __restrict__ meta,
                   const unsigned char* __restrict__ shapes, const int4* __restrict__ k0,
                   const int32_t* __restrict__ krows, int64_t n_strip, int stride, int off_pos, int sh_stride,
                   int off_prow, int off_ent, unsigned long long* __restrict__ ticket,
                   double* __restrict__ values) {
    constexpr int P = kStripElems, KB = P * 128;
    extern __shared__ __align__(16) unsigned char smem_st[];
    const int tid = threadIdx.x;
    const int slot = KB + stride + sh_stride;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_st + STAGES * slot);
    int64_t* s_q = reinterpret_cast<int64_t*>(bars + STAGES);  // 8 claimed strips, issue -> compute
    const int64_t G = gridDim.x;
    int64_t t_next = 0;  // thread 0: the ticket after the one being issued (round trip off the issue path)
    auto claim = [&]() -> int64_t {
        const int64_t r = t_next;
        t_next = ticket ? static_cast<int64_t>(atomicAdd(ticket, 1ull)) : r + G;
        return r;
    };
    auto issue = [&](int stage, int64_t st) {  // thread 0
        const uint32_t bar = smem_u32(bars + stage);
        if (st >= n_strip) {
            mbar_arrive(bar);
            return;
        }
        unsigned char* sb = smem_st + stage * slot;
        fence_proxy_async_smem();  // the stage was last read by generic loads
        const int4 kk = __ldg(k0 + st);
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(kk.y * 128 + stride + sh_stride));
        if (kk.x >= 0) {
            bulk_g2s(smem_u32(sb), K + static_cast<int64_t>(kk.x) * 16, static_cast<uint32_t>(kk.y * 128), bar);
        } else {
            for (int k = 0; k < kk.y; ++k)
                bulk_g2s(smem_u32(sb + k * 128), K + static_cast<int64_t>(__ldg(krows + st * P + k)) * 16, 128u, bar);
        }
        bulk_g2s(smem_u32(sb + KB), meta + st * stride, static_cast<uint32_t>(stride), bar);
        bulk_g2s(smem_u32(sb + KB + stride), shapes + static_cast<int64_t>(kk.z) * sh_stride,
                 static_cast<uint32_t>(sh_stride), bar);
    };
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) mbar_init(smem_u32(bars + st), 1);
        mbar_fence_init();
        t_next = ticket ? static_cast<int64_t>(atomicAdd(ticket, 1ull)) : static_cast<int64_t>(blockIdx.x);
        for (int j = 0; j < STAGES - 1; ++j) {
            const int64_t st = claim();
            s_q[j & 7] = st;
            issue(j, st);
        }
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
        const int64_t st = s_q[it & 7];
        if (st >= n_strip) break;  // claims only grow: every later one is past the end too
        const int stage = it % STAGES;
        if (tid == 0) {  // refill the stage the previous iteration released (barrier below)
            const int j = it + STAGES - 1;
            const int64_t sn = claim();
            s_q[j & 7] = sn;
            issue(j % STAGES, sn);
        }
        mbar_wait(smem_u32(bars + stage), (phase >> stage) & 1u);
        phase ^= 1u << stage;
        const unsigned char* sb = smem_st + stage * slot;
        const unsigned char* mb = sb + KB;
        const unsigned char* hb = mb + stride;
        const int n_pairs = *reinterpret_cast<const int*>(mb);
        const int64_t* rows = reinterpret_cast<const int64_t*>(mb + 16);
        const uint8_t* ppos = mb + off_pos;
        const uint16_t* pend = reinterpret_cast<const uint16_t*>(hb);
        const uint8_t* prow = hb + off_prow;
        const uint16_t* ent = reinterpret_cast<const uint16_t*>(hb + off_ent);
        const double* Ks = reinterpret_cast<const double*>(sb);
        for (int t = tid; t < n_pairs; t += kStripThreads) {
            const int b = t ? pend[t - 1] : 0, e = pend[t];
            double sum = 0.0;
            for (int i = b; i < e; ++i) sum += Ks[ent[i]];
            FEA_DCHECK(prow[t] < reinterpret_cast<const int*>(mb)[2] && rows[prow[t]] >= 0);
            atomicAdd(values + rows[prow[t]] + ppos[t], sum);
        }
        __syncthreads();
    }
}

// --- launch helpers --------------------------------------------------------

// Per (plan, kernel, block size, shared memory): raise the kernel's dynamic shared-memory
// limit if needed and return its resident CTAs per SM. Cached in the plan, so a repeated
// assembly does no attribute or occupancy queries (host latency on small meshes).
template <class F>
int launch_prep(fea_plan* p, F* kern, int threads, size_t smem) {
    const void* fn = reinterpret_cast<const void*>(kern);
    for (const auto& c : p->occ_cache)
        if (c.fn == fn && c.smem == smem && c.threads == threads) return c.per_sm;
    if (smem > 48 * 1024) {
        // the attribute is per kernel and process-wide: only ever raise it (another plan may
        // need more than this one)
        static std::mutex mu;
        static std::vector<std::pair<std::pair<const void*, int>, size_t>> limit;
        std::lock_guard<std::mutex> lk(mu);
        size_t* cur = nullptr;
        for (auto& l : limit)
            if (l.first.first == fn && l.first.second == p->device) cur = &l.second;
        if (!cur || *cur < smem) {
            FEA_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            if (cur) *cur = smem;
            else limit.push_back({{fn, p->device}, smem});
        }
    }
    int per_sm = 0;
    FEA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    p->occ_cache.push_back({fn, smem, threads, per_sm});
    return per_sm;
}

#ifndef FEA_PDL
#define FEA_PDL 1
#endif
// Launch with the programmatic-dependent-launch attribute (FEA_PDL): back-to-back assemblies on
// one stream (or in a CUDA graph) overlap the next kernel's launch and metadata prologue with
// the previous kernel's tail. Kernels launched this way call pdl_wait() before K / values.
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, Args... args) {
    if (!FEA_PDL) {
        kern<<<grid, block, smem, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FEA_CK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// Traversal window of a windowed gather launch (fea_plan::win_t0 / win_n).
struct Win {
    int64_t t0, n;
};
inline Win window_of(const fea_plan* p) {
    return p->win_n >= 0 ? Win{p->win_t0, p->win_n} : Win{0, p->n_own};
}
// Launchers whose kernel does not take windows: report it to a query, refuse a window.
inline bool no_window(fea_plan* p) {
    if (p->win_query) {
        p->win_ok = false;
        return true;
    }
    FEA_REQUIRE(p->win_n < 0, FEA_ERR_INVALID, "internal: traversal window on a kernel without windows");
    return false;
}

GenK gen_of(const fea_plan* p) {
    GenK g{};
    g.on = p->gen_on ? 1 : 0;
    g.seed = p->gen_seed;
    g.ids = (p->k_compact && p->partitioned) ? p->elem_id.as<int64_t>() : nullptr;
    return g;
}

template <int G, int R, int PF, class PosT>
void run_gather_stream(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                       cudaStream_t s) {
    constexpr int GPW = 32 / G;
    const int acc_stride = p->d * p->d * p->max_cnt + 1;  // +1 staggers groups across banks
    constexpr int kBlk = blk_of<G>();
    const int pw_blk = kBlk * p->pstride * static_cast<int>(sizeof(PosT)) / 4;
    FEA_FITS((pw_blk + G - 1) / G <= kPosW);
    const size_t smem = static_cast<size_t>(kWarps) * GPW *
                        (acc_stride * sizeof(double) + 2 * (kBlk + pw_blk) * sizeof(int32_t));
    FEA_FITS(smem <= 227 * 1024);
    auto kern = p->dup_nodes ? k_gather_stream<G, R, PF, PosT, false> : k_gather_stream<G, R, PF, PosT, true>;
    const int occ = launch_prep(p, kern, kWarps * 32, smem);
    const int n_sm = p->sms;
    if (no_window(p) || p->n_own == 0) return;
    // persistent: one wave of CTAs, each group a contiguous node range (>= 2 nodes per group)
    int64_t blocks = static_cast<int64_t>(std::max(occ, 1)) * n_sm;
    blocks = std::min<int64_t>(blocks, (p->n_own + 2 * kWarps * GPW - 1) / (2 * kWarps * GPW));
    blocks = std::max<int64_t>(blocks, 1);
    const int64_t n_groups = blocks * kWarps * GPW;
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        K, p->adj_ptr.as<int64_t>(), in.adj, static_cast<const PosT*>(in.posA), p->nptr.as<int64_t>(),
        p->n_own, n_groups, p->d, p->npe, p->pstride, acc_stride, accumulate ? 1 : 0, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

template <int G, int R, int PF, class PosT>
void run_gather_node(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                     cudaStream_t s) {
    constexpr int GPW = 32 / G;
    const int acc_stride = p->d * p->d * p->max_cnt + 1;  // +1 staggers groups across banks
    const int pos_stride = static_cast<int>((std::max<int64_t>(p->max_adj, 1) * p->pstride + 7) & ~int64_t(7));
    size_t smem = static_cast<size_t>(kWarps) * GPW *
                  (acc_stride * sizeof(double) + pos_stride * sizeof(PosT));
    FEA_FITS(smem <= 227 * 1024);
    auto kern = p->gen_on ? (p->dup_nodes ? k_gather_node<G, R, PF, PosT, false, true>
                                          : k_gather_node<G, R, PF, PosT, true, true>)
                          : (p->dup_nodes ? k_gather_node<G, R, PF, PosT, false, false>
                                          : k_gather_node<G, R, PF, PosT, true, false>);
    launch_prep(p, kern, kWarps * 32, smem);
    if (no_window(p)) return;
    const int64_t groups = p->n_own;
    const int64_t blocks = (groups + kWarps * GPW - 1) / (kWarps * GPW);
    if (blocks == 0) return;
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        K, p->adj_ptr.as<int64_t>(), in.adj, static_cast<const PosT*>(in.posA),
        p->nptr.as<int64_t>(), p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->n_own, p->d,
        p->npe, p->pstride, acc_stride, pos_stride, accumulate ? 1 : 0, p->d * p->m * 8 < 128 ? 1 : 0,
        gen_of(p), values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

// Kernel choice (measured): one lane group per warp (G == 32, large element
// blocks) streams persistently; smaller blocks run one node per lane group, many warps.
template <int G, int R, int PF, class PosT>
void run_gather(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                cudaStream_t s) {
    if (G == 32 && R >= 8 && !p->node_order.p && !p->gen_on) run_gather_stream<G, R, PF, PosT>(p, in, K, values, accumulate, s);
    else run_gather_node<G, R, PF, PosT>(p, in, K, values, accumulate, s);
}

template <int D, int NPE>
void run_gather_slot(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                     cudaStream_t s) {
    const int dm = D * D * NPE;
    const int nbuf = static_cast<int>(std::max<int64_t>(p->max_adj, 1));
#ifndef FEA_SLOT_TIGHT_INV
#define FEA_SLOT_TIGHT_INV 0
#endif
    // inverse-table row: 32 bytes, or (FEA_SLOT_TIGHT_INV) the longest node row rounded to 4
    // bytes: on hex8 (27 column nodes) 28 bytes per block bring a 4-warp CTA to 37,824 B and 6
    // CTAs per SM instead of 5 — faster only when the clock is power-capped (bench 0.292 vs
    // 0.305 ms at ~1,610-1,680 MHz), slower at full clock (0.312 vs 0.280 ms at 1,965 MHz;
    // cfg5 20.9 vs 17.6 ms), like 8-warp CTAs: not the default
    const int istr = FEA_SLOT_TIGHT_INV ? std::max(4, (p->max_cnt + 3) & ~3) : 32;
    const size_t smem = static_cast<size_t>(kSlotWarps) * nbuf * (2 * dm * sizeof(double) + istr) + kSlotWarps * 16;
    // fixed-stride metadata table per incidence order (lazily; 16 + 16 * nbuf bytes per node)
    const bool sorted_inc = in.adj == p->adj.as<int32_t>();
    feagpu::DevBuf& fx = sorted_inc ? p->slot_rec : p->slot_recC;
    const bool fixed = !p->gen_on && (sorted_inc || in.adj == p->adjC.as<int32_t>()) &&
                       !p->kn.slot_no_fixed && (fx.p || !capturing(s));
    if (fixed && !fx.p) {
        if (!p->slot_hdr.p) p->slot_hdr.alloc(std::max<int64_t>(p->n_own, 1) * 16);
        fx.alloc(std::max<int64_t>(p->n_own, 1) * nbuf * 16);
        k_slot_fixed_build<<<grid_for(p->n_own * 32, 256), 256, 0, s>>>(
            p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->adj_ptr.as<int64_t>(), in.adj,
            static_cast<const uint32_t*>(in.posA), p->nptr.as<int64_t>(), p->n_own, nbuf, NPE <= 4 ? 1 : 2,
            p->slot_hdr.as<int4>(), fx.as<int4>());
        FEA_CK(cudaGetLastError());
    }
    auto kern = fixed ? (p->dup_nodes ? k_gather_slot<D, NPE, false, false, true> : k_gather_slot<D, NPE, true, false, true>)
                : p->gen_on ? (p->dup_nodes ? k_gather_slot<D, NPE, false, true, false> : k_gather_slot<D, NPE, true, true, false>)
                          : (p->dup_nodes ? k_gather_slot<D, NPE, false, false, false> : k_gather_slot<D, NPE, true, false, false>);
    const int per_sm = launch_prep(p, kern, kSlotWarps * 32, smem);
    if (p->win_query) {
        p->win_ok = true;
        return;
    }
    // window: shift the per-traversal-position arrays (order, fixed tables; without an order
    // the node id is the position, so adj_ptr / nptr shift instead)
    const Win wn = window_of(p);
    const int32_t* order = p->node_order.p ? p->node_order.as<int32_t>() + wn.t0 : nullptr;
    const int64_t shift = order ? 0 : wn.t0;
    const int64_t want = (wn.n + kSlotWarps - 1) / kSlotWarps;  // one node per warp at most
    const int64_t blocks = std::min<int64_t>(want, static_cast<int64_t>(p->sms) * std::max(per_sm, 1));
    if (blocks == 0) return;
    kern<<<static_cast<unsigned>(blocks), kSlotWarps * 32, smem, s>>>(
        K, p->adj_ptr.as<int64_t>() + shift, in.adj, static_cast<const uint8_t*>(in.posA),
        p->nptr.as<int64_t>() + shift, order, wn.n, nbuf, istr, accumulate ? 1 : 0, gen_of(p),
        fixed ? p->slot_hdr.as<int4>() + wn.t0 : nullptr, fixed ? fx.as<int4>() + wn.t0 * nbuf : nullptr, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

// lane = slot kernel applies: d in {2,3,4}, element rows of <= 8 nodes with byte positions,
// node rows of <= 32 column nodes, <= 32 incidences per node, 16-byte chunks, <= 24 KB smem per warp
bool slot_applies(const fea_plan* p) {
    if (p->d < 2 || p->d > 4 || (p->npe != 4 && p->npe != 8) || p->pos_bytes != 1 || p->max_cnt > 32 ||
        p->max_adj > 32 || p->gen_on)
        return false;
    const int64_t dm = static_cast<int64_t>(p->d) * p->d * p->npe;
    if (dm % 2) return false;
    return 2 * std::max<int64_t>(p->max_adj, 1) * dm * 8 <= 24 * 1024;  // per-warp double buffer
}

#ifndef FEA_CN_PF8
#define FEA_CN_PF8 2
#endif
// largest per-CTA sum of node blocks (+1 stagger each) over CTAs of `per_cta` consecutive
// traversal nodes: the packed accumulator size of k_gather_cn
__global__ void k_cta_acc_max(const int32_t* __restrict__ order, const int64_t* __restrict__ nptr,
                              int64_t n_own, int dd, int per_cta, unsigned long long* out) {
    const int64_t n_cta = (n_own + per_cta - 1) / per_cta;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cta;
         c += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long sum = 0;
        for (int g = 0; g < per_cta; ++g) {
            const int64_t t = c * per_cta + g;
            if (t >= n_own) break;
            const int64_t u = order != nullptr ? order[t] : t;
            sum += static_cast<unsigned long long>(dd * (nptr[u + 1] - nptr[u]) + 1);
        }
        atomicMax(out, sum);
    }
}

int64_t cn_cta_acc(fea_plan* p, int per_cta, cudaStream_t s) {
    if (p->kn.cn_unpacked) return static_cast<int64_t>(per_cta) * (p->d * p->d * p->max_cnt + 1);
    if (p->cn_cta_acc > 0 && p->cn_cta_per == per_cta) return p->cn_cta_acc;
    DevBuf out;
    out.alloc(8);
    FEA_CK(cudaMemsetAsync(out.p, 0, 8, s));
    if (p->n_own > 0) {
        k_cta_acc_max<<<grid_for((p->n_own + per_cta - 1) / per_cta, 256), 256, 0, s>>>(
            p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->nptr.as<int64_t>(), p->n_own,
            p->d * p->d, per_cta, out.as<unsigned long long>());
        FEA_CK(cudaGetLastError());
    }
    unsigned long long v = 0;
    FEA_CK(cudaMemcpyAsync(&v, out.p, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    p->cn_cta_acc = std::max<int64_t>(static_cast<int64_t>(v), 1);
    p->cn_cta_per = per_cta;
    return p->cn_cta_acc;
}

template <int G, int D, int PF, class PosT>
void run_gather_cn(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                   cudaStream_t s) {
    constexpr int GPW = 32 / G;
    const int acc_stride = p->d * p->d * p->max_cnt + 1;  // +1 staggers groups across banks (swept: 1-2 best)
    const int pos_stride = static_cast<int>((std::max<int64_t>(p->max_adj, 1) * p->pstride + 7) & ~int64_t(7));
    const int64_t cta_acc = cn_cta_acc(p, kWarps * GPW, s);
    const size_t smem = static_cast<size_t>(cta_acc) * sizeof(double) +
                        static_cast<size_t>(kWarps) * GPW * pos_stride * sizeof(PosT);
    FEA_FITS(smem <= 227 * 1024);
    if (G == 32 && sizeof(PosT) == 1 && !p->dup_nodes && p->max_adj <= kCnrSlots &&
        p->npe <= kCnrBytes - 4 && (in.adj == p->adj.as<int32_t>() || in.adj == p->adjC.as<int32_t>()) &&
        !p->kn.cn_no_records &&
        ((p->cnr_hdr.p && (in.adj == p->adj.as<int32_t>() ? p->cnr_rec.p : p->cnr_recC.p)) || !capturing(s))) {
        // built lazily on the first assembly of each incidence order: 16 + 256 bytes per node
        feagpu::DevBuf& recs = in.adj == p->adj.as<int32_t>() ? p->cnr_rec : p->cnr_recC;
        if (!p->cnr_hdr.p || !recs.p) {
            if (!p->cnr_hdr.p) p->cnr_hdr.alloc(std::max<int64_t>(p->n_own, 1) * 16);
            recs.alloc(std::max<int64_t>(p->n_own, 1) * kCnrSlots * kCnrBytes);
            if (p->n_own > 0) {
                k_cnr_build<<<grid_for(p->n_own, 256), 256, 0, s>>>(
                    p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->adj_ptr.as<int64_t>(), in.adj,
                    static_cast<const uint8_t*>(in.posA), p->nptr.as<int64_t>(), p->n_own, p->npe, p->pstride,
                    p->d, kWarps, p->cnr_hdr.as<int4>(), recs.as<int32_t>());
                FEA_CK(cudaGetLastError());
            }
        }
        const size_t smem_r = static_cast<size_t>(cta_acc) * sizeof(double) + kWarps * kCnrSlots * kCnrBytes;
        FEA_FITS(smem_r <= 227 * 1024);
        auto kr = p->gen_on ? k_gather_cnr<D, FEA_CNR_PF, true> : k_gather_cnr<D, FEA_CNR_PF, false>;
        launch_prep(p, kr, kWarps * 32, smem_r);
        if (p->win_query) {
            p->win_ok = true;
            return;
        }
        // windows start at multiples of kWarps (the headers' packed accumulator offsets are
        // relative to CTAs of kWarps consecutive traversal positions)
        const Win wn = window_of(p);
        FEA_REQUIRE(wn.t0 % kWarps == 0, FEA_ERR_INVALID, "internal: window not CTA-aligned");
        const int64_t blocks_r = (wn.n + kWarps - 1) / kWarps;
        if (blocks_r == 0) return;
        kr<<<static_cast<unsigned>(blocks_r), kWarps * 32, smem_r, s>>>(
            K, p->cnr_hdr.as<int4>() + wn.t0, recs.as<int2>() + wn.t0 * (kCnrSlots * kCnrBytes / 8), wn.n, p->npe,
            accumulate ? 1 : 0, cta_acc, gen_of(p), values);
        FEA_CK(cudaGetLastError());
        p->last_launches += 1;
        return;
    }
    auto kern = p->gen_on ? (p->dup_nodes ? k_gather_cn<G, D, PF, PosT, false, true>
                                          : k_gather_cn<G, D, PF, PosT, true, true>)
                          : (p->dup_nodes ? k_gather_cn<G, D, PF, PosT, false, false>
                                          : k_gather_cn<G, D, PF, PosT, true, false>);
    launch_prep(p, kern, kWarps * 32, smem);
    if (no_window(p)) return;
    const int64_t blocks = (p->n_own + kWarps * GPW - 1) / (kWarps * GPW);
    if (blocks == 0) return;
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        K, p->adj_ptr.as<int64_t>(), in.adj, static_cast<const PosT*>(in.posA), p->nptr.as<int64_t>(),
        p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->n_own, p->npe, p->pstride, acc_stride,
        pos_stride, accumulate ? 1 : 0, gen_of(p), cta_acc, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

template <int G, int PF, class PosT>
void run_gather_d1(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                   cudaStream_t s) {
    constexpr int GPW = 32 / G;
    // accumulator stride = 3 (mod 16 doubles): swept all odd residues on cfg3, 3 fewest conflicts
    // (0.642 ms vs 0.664 at 15 and 0.670 at 1)
    int acc_stride = std::max(p->max_cnt, 1);
    int acc_mod = 3;
    if (p->kn.d1_acc_mod >= 0) acc_mod = p->kn.d1_acc_mod;
    while ((acc_stride & 15) != acc_mod) ++acc_stride;
    const int cap = static_cast<int>(std::max<int64_t>(p->max_adj, 1));
    const int pw = p->pstride * static_cast<int>(sizeof(PosT)) / 4;
    const int rw = pw == 1 ? 2 : (pw + 4) & ~3;
    // per-group record stride in words with stride/2 odd: the 8 groups' 8-byte record reads
    // of one step land on 8 distinct bank pairs
    int rec_stride = cap * rw;
    if (((rec_stride / 2) & 1) == 0) rec_stride += 2;
    const size_t smem = static_cast<size_t>(kWarps) * GPW *
                        (acc_stride * sizeof(double) + static_cast<size_t>(rec_stride) * sizeof(int32_t));
    FEA_FITS(smem <= 227 * 1024);
    auto kern = p->gen_on ? (p->dup_nodes ? k_gather_d1<G, PF, PosT, false, true> : k_gather_d1<G, PF, PosT, true, true>)
                          : (p->dup_nodes ? k_gather_d1<G, PF, PosT, false, false> : k_gather_d1<G, PF, PosT, true, false>);
    const int64_t per_cta = static_cast<int64_t>(kWarps) * GPW;
    const int64_t blocks = (p->n_own + per_cta - 1) / per_cta;
    if (blocks == 0) return;
    // traversal-ordered records: sorted incidences (trav_rec) or colour-ordered ones (trav_recC)
    const DevBuf& recs = in.adj == p->adj.as<int32_t>() ? p->trav_rec : p->trav_recC;
    const bool trav = recs.p != nullptr && (in.adj == p->adj.as<int32_t>() || in.adj == p->adjC.as<int32_t>());
    FEA_REQUIRE(!trav || p->trav_rw == rw, FEA_ERR_INVALID, "traversal record width mismatch");
    // lane-owned slots (the plan coloured every node's star with 4 lanes)
    if (G == 4 && p->npe == 4 && trav && rw == 2 && !p->dup_nodes && sizeof(PosT) == 1 && !p->gen_on &&
        p->ln_ok && !p->kn.d1_no_lane) {
        const DevBuf& lrecs = in.adj == p->adj.as<int32_t>() ? p->ln_rec : p->ln_recC;
        FEA_REQUIRE(lrecs.p != nullptr, FEA_ERR_INVALID, "lane records missing");
        const Win wn = window_of(p);
        {
            void (*ks)(const double*, int64_t, int, const int4*, const void*, int, int, int, int, double*) =
                p->ln_rec4 ? k_gather_d1s<FEA_D1S_U, true> : k_gather_d1s<FEA_D1S_U, false>;
            const size_t smems = static_cast<size_t>(p->ln_q) * kD1sThreads * sizeof(double);
            launch_prep(p, ks, kD1sThreads, smems);
            if (p->win_query) {
                p->win_ok = true;
                return;
            }
            const int64_t blocks_s = (wn.n + kD1sThreads / 4 - 1) / (kD1sThreads / 4);
            if (blocks_s == 0) return;
            launch_pdl(ks, static_cast<unsigned>(blocks_s), kD1sThreads, smems, s, K, wn.n, accumulate ? 1 : 0,
                       p->ln_hdr.as<int4>() + 2 * wn.t0, static_cast<const void*>(lrecs.p), p->ln_q, p->ln_wq[0],
                       p->ln_wq[1], p->ln_wq[2], values);
            FEA_CK(cudaGetLastError());
            p->last_launches += 1;
            return;
        }
    }
    // npe = 4 with traversal records: direct-record kernel for a materialized K, two-lane
    // kernel for the fused supplier
    if (G == 4 && p->npe == 4 && trav && rw == 2 && !p->dup_nodes && sizeof(PosT) == 1 && !p->gen_on &&
        !p->kn.d1_no_direct) {
        const size_t smemg = static_cast<size_t>(kWarps) * GPW * acc_stride * sizeof(double);
        auto kg = k_gather_d1g<FEA_D1G_U>;
        launch_prep(p, kg, kWarps * 32, smemg);
        if (p->win_query) {
            p->win_ok = true;
            return;
        }
        const Win wn = window_of(p);
        const int64_t blocks_w = (wn.n + per_cta - 1) / per_cta;
        if (blocks_w == 0) return;
        launch_pdl(kg, static_cast<unsigned>(blocks_w), kWarps * 32, smemg, s, K, wn.n, acc_stride,
                   accumulate ? 1 : 0, p->trav_ptr.as<int64_t>() + wn.t0, p->trav_meta.as<int64_t>() + wn.t0,
                   reinterpret_cast<const int2*>(recs.as<int32_t>()), values);
        FEA_CK(cudaGetLastError());
        p->last_launches += 1;
        return;
    }
    if (G == 4 && p->npe == 4 && trav && rw == 2 && !p->dup_nodes && sizeof(PosT) == 1 && p->gen_on &&
        !p->kn.d1_no_vec) {
        constexpr int GPW2 = 16;
        int acc_stride2 = std::max(p->max_cnt, 1);
        int acc_mod2 = 3;
        if (p->kn.d1v_acc_mod >= 0) acc_mod2 = p->kn.d1v_acc_mod;
        while ((acc_stride2 & 15) != acc_mod2) ++acc_stride2;
        const size_t smem2 = static_cast<size_t>(kWarps) * GPW2 *
                             (acc_stride2 * sizeof(double) + static_cast<size_t>(rec_stride) * sizeof(int32_t));
        FEA_FITS(smem2 <= 227 * 1024);
#ifndef FEA_D1V_PF
#define FEA_D1V_PF 4
#endif
        auto kern2 = k_gather_d1v<FEA_D1V_PF>;
        launch_prep(p, kern2, kWarps * 32, smem2);
        if (no_window(p)) return;
        const int64_t per_cta2 = static_cast<int64_t>(kWarps) * GPW2;
        const int64_t blocks2 = (p->n_own + per_cta2 - 1) / per_cta2;
        if (blocks2 == 0) return;
        kern2<<<static_cast<unsigned>(blocks2), kWarps * 32, smem2, s>>>(
            p->n_own, cap, rec_stride, acc_stride2, accumulate ? 1 : 0, p->trav_ptr.as<int64_t>(), p->trav_meta.as<int64_t>(), recs.as<int32_t>(), gen_of(p), values);
        FEA_CK(cudaGetLastError());
        p->last_launches += 1;
        return;
    }
    launch_prep(p, kern, kWarps * 32, smem);
    if (no_window(p)) return;
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        K, p->adj_ptr.as<int64_t>(), in.adj, static_cast<const PosT*>(in.posA), p->nptr.as<int64_t>(),
        p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->n_own, p->npe, p->pstride, cap,
        rec_stride, acc_stride, accumulate ? 1 : 0, p->m * 8 < 128 ? 1 : 0, trav ? p->trav_ptr.as<int64_t>() : nullptr,
        trav ? p->trav_meta.as<int64_t>() : nullptr, trav ? recs.as<int32_t>() : nullptr, gen_of(p), values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

// Deterministic routes without a shared-memory accumulator, for plans whose largest node row
// block fits none of the kernels above: a warp owns a node and folds the node's incident row
// blocks, in incidence order, straight into the node's block of the values array (nobody else
// writes it; __syncwarp orders the lanes' reads and writes between incidences). Without repeated
// nodes the entries of one incidence hit distinct slots and are spread over the lanes; with
// repeated nodes the columns go one after the other, as scatter_element's loop does. Per slot a
// left fold from the start value in incidence order: the bits of the kernels above.
template <class PosT>
__global__ void __launch_bounds__(256)
    k_gather_global(const double* __restrict__ K, const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj,
                    const PosT* __restrict__ posA, const int64_t* __restrict__ nptr, int64_t n_own, int d, int npe,
                    int pstride, int accumulate, int dup_nodes, GenK gen, double* values) {
    const int lane = threadIdx.x & 31;
    const int dd = d * d, m = d * npe;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n_own;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b0 = adj_ptr[v], c0 = nptr[v];
        const int n = static_cast<int>(adj_ptr[v + 1] - b0);
        const int64_t rowlen = static_cast<int64_t>(d) * (nptr[v + 1] - c0);
        double* blk = values + static_cast<int64_t>(dd) * c0;
        if (!accumulate)
            for (int64_t i = lane; i < d * rowlen; i += 32) blk[i] = 0.0;
        __syncwarp();
        for (int k = 0; k < n; ++k) {
            const int32_t entry = adj[b0 + k];
            const int64_t krow = entry / npe;
            const int a = static_cast<int>(entry - krow * npe);
            const double* src = K + static_cast<int64_t>(entry) * d * m;
            const uint64_t he = gen.on ? kgen_elem(gen.seed, gen.ids ? gen.ids[krow] : krow) : 0;
            const PosT* pos = posA + (b0 + k) * pstride;
            auto add = [&](int b, int t) {
                const int ki = t / d, kj = t - ki * d;
                const double x = gen.on ? kgen_entry(he, a * d + ki, b * d + kj) : src[ki * m + b * d + kj];
                FEA_DCHECK(static_cast<int64_t>(pos[b]) * d + kj < rowlen);
                double* dst = blk + ki * rowlen + static_cast<int64_t>(pos[b]) * d + kj;
                *dst += x;
            };
            if (!dup_nodes) {
                for (int t = lane; t < npe * dd; t += 32) add(t / dd, t % dd);
                __syncwarp();
            } else {
                for (int b = 0; b < npe; ++b) {
                    for (int t = lane; t < dd; t += 32) add(b, t);
                    __syncwarp();
                }
            }
        }
    }
}

template <class PosT>
void run_gather_global(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                       cudaStream_t s) {
    if (no_window(p) || p->n_own == 0) return;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((p->n_own + 7) / 8, static_cast<int64_t>(p->sms) * 8));
    k_gather_global<PosT><<<blocks, 256, 0, s>>>(K, p->adj_ptr.as<int64_t>(), in.adj, static_cast<const PosT*>(in.posA),
                                                 p->nptr.as<int64_t>(), p->n_own, p->d, p->npe, p->pstride,
                                                 accumulate ? 1 : 0, p->dup_nodes ? 1 : 0, gen_of(p), values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

template <class PosT>
void gather_fitting(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate, cudaStream_t s);

template <class PosT>
void gather(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
            cudaStream_t s) {
    if (!p->gather_global && !p->kn.gather_global) {
        try {
            return gather_fitting<PosT>(p, in, K, values, accumulate, s);
        } catch (const DoesNotFit&) {
            p->gather_global = true;  // the checks precede every launch: nothing has run yet
        }
    }
    run_gather_global<PosT>(p, in, K, values, accumulate, s);
}

template <class PosT>
void gather_fitting(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                    cudaStream_t s) {
    const int dm = p->d * p->m;
    // lane = column node (d in {2,3,4}, npe <= 32); measured faster than the decode-table
    // kernels for every such shape
    // d = 1: staged-stream kernel
    if (!p->d1_disabled && p->d == 1 && p->npe <= 32) {
#ifndef FEA_D1_PF
#define FEA_D1_PF 4  // swept 2-12 on cfg3: 3-4 best
#endif
        if (p->npe <= 4) return run_gather_d1<4, FEA_D1_PF, PosT>(p, in, K, values, accumulate, s);
        if (p->npe <= 8) return run_gather_d1<8, FEA_D1_PF, PosT>(p, in, K, values, accumulate, s);
        if (p->npe <= 16) return run_gather_d1<16, 4, PosT>(p, in, K, values, accumulate, s);
        return run_gather_d1<32, 4, PosT>(p, in, K, values, accumulate, s);
    }
    // (bulk copies need 16-byte aligned element matrices)
    if (!p->slot_disabled && slot_applies(p) && (reinterpret_cast<uintptr_t>(K) & 15) == 0) {
        const bool n4 = p->npe == 4;
        switch (p->d) {
            case 2: return n4 ? run_gather_slot<2, 4>(p, in, K, values, accumulate, s) : run_gather_slot<2, 8>(p, in, K, values, accumulate, s);
            case 3: return n4 ? run_gather_slot<3, 4>(p, in, K, values, accumulate, s) : run_gather_slot<3, 8>(p, in, K, values, accumulate, s);
            default: return n4 ? run_gather_slot<4, 4>(p, in, K, values, accumulate, s) : run_gather_slot<4, 8>(p, in, K, values, accumulate, s);
        }
    }
    if (!p->cn_disabled && p->d >= 2 && p->d <= 4 && p->npe <= 32) {
        const int G = p->npe <= 4 ? 4 : p->npe <= 8 ? 8 : p->npe <= 16 ? 16 : 32;
        switch (G * 10 + p->d) {
            case 42: return run_gather_cn<4, 2, 2, PosT>(p, in, K, values, accumulate, s);
            case 43: return run_gather_cn<4, 3, 2, PosT>(p, in, K, values, accumulate, s);
            case 44: return run_gather_cn<4, 4, 2, PosT>(p, in, K, values, accumulate, s);
            case 82: return run_gather_cn<8, 2, 2, PosT>(p, in, K, values, accumulate, s);
            case 83: return run_gather_cn<8, 3, FEA_CN_PF8, PosT>(p, in, K, values, accumulate, s);
            case 84: return run_gather_cn<8, 4, 2, PosT>(p, in, K, values, accumulate, s);
            case 163: return run_gather_cn<16, 3, 2, PosT>(p, in, K, values, accumulate, s);
#ifndef FEA_CN_PF32
#define FEA_CN_PF32 2  // swept on hex27 (cfg4), packed accumulators: PF 1 (64 regs, 7 CTAs/SM) 1.99 ms, PF 2 (80 regs, 6) 1.95, PF 2 at 72 regs 2.06, PF 3 spills
#endif
            case 323: return run_gather_cn<32, 3, FEA_CN_PF32, PosT>(p, in, K, values, accumulate, s);
            default: break;
        }
    }
    if (dm <= 4) run_gather<4, 1, 8, PosT>(p, in, K, values, accumulate, s);
    else if (dm <= 8) run_gather<8, 1, 8, PosT>(p, in, K, values, accumulate, s);
    else if (dm <= 16) run_gather<16, 1, 4, PosT>(p, in, K, values, accumulate, s);
    else if (dm <= 32) run_gather<32, 1, 4, PosT>(p, in, K, values, accumulate, s);
#ifndef FEA_HEX8_PF
#define FEA_HEX8_PF 2
#endif
    else if (dm == 72) run_gather<8, 9, FEA_HEX8_PF, PosT>(p, in, K, values, accumulate, s);
    else if (dm <= 128) run_gather<32, 4, 2, PosT>(p, in, K, values, accumulate, s);
    else if (dm <= 256) run_gather<32, 8, 2, PosT>(p, in, K, values, accumulate, s);
    else if (dm <= 512) run_gather<32, 16, 1, PosT>(p, in, K, values, accumulate, s);
    else throw DoesNotFit{};
}

template <int G, class PosT, bool ATOMIC>
void run_scatter(fea_plan* p, const double* K, const int32_t* list, int64_t n_list, double* values,
                 cudaStream_t s) {
    if (n_list == 0) return;
    constexpr int GPW = 32 / G;
    const int mm = p->m * p->m;
    const size_t smem = static_cast<size_t>((mm + 1) & ~1) * 4 +
                        static_cast<size_t>(kWarps) * GPW * p->npe * (8 + 4);
    FEA_REQUIRE(smem <= 227 * 1024, FEA_ERR_INVALID, "element matrix too large for the scatter kernel");
    auto kern = k_scatter<G, PosT, ATOMIC>;
    launch_prep(p, kern, kWarps * 32, smem);
    const int64_t blocks = std::min<int64_t>((n_list + kWarps * GPW - 1) / (kWarps * GPW), 148 * 16);
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        K, list, n_list, p->elem_krow.as<int32_t>(), p->conn_k.as<int32_t>(), p->posE.as<PosT>(),
        p->nptr.as<int64_t>(), p->node_begin, p->n_own, p->d, p->npe, p->dup_nodes ? 1 : 0, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

template <class PosT, bool ATOMIC>
void scatter(fea_plan* p, const double* K, const int32_t* list, int64_t n_list, double* values,
             cudaStream_t s) {
    const int mm = p->m * p->m;
    if (mm <= 4) run_scatter<4, PosT, ATOMIC>(p, K, list, n_list, values, s);
    else if (mm <= 8) run_scatter<8, PosT, ATOMIC>(p, K, list, n_list, values, s);
    else if (mm <= 16) run_scatter<16, PosT, ATOMIC>(p, K, list, n_list, values, s);
    else run_scatter<32, PosT, ATOMIC>(p, K, list, n_list, values, s);
}

template <int D, int NPE, class PosT>
void run_atomic_staged(fea_plan* p, const double* K, double* values, cudaStream_t s) {
    using S = AtomicShape<D, NPE, PosT>;
    constexpr int STAGES = FEA_AT_STAGES;
    const int64_t n_steps = p->at_E_pad / S::B;
    if (n_steps == 0) return;
    const size_t smem = static_cast<size_t>(kWarps) * STAGES * S::STAGE;
    auto kern = k_atomic_staged<D, NPE, PosT, STAGES>;
    const int per_sm = launch_prep(p, kern, kWarps * 32, smem);
    const int sms = p->sms;
    const int64_t blocks = std::min<int64_t>((n_steps + kWarps - 1) / kWarps,
                                             static_cast<int64_t>(sms) * std::max(per_sm, 1));
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        K, p->at_krow.as<int32_t>(), p->at_rows.as<int64_t>(), p->at_pos.as<PosT>(), n_steps, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

template <int D, int NPE, class PosT>
void run_atomic_cta(fea_plan* p, const double* K, double* values, cudaStream_t s) {
    const int64_t n_steps = p->at_E_pad;
    if (n_steps == 0) return;
    auto kern = k_atomic_direct<D, NPE, PosT>;
    const int per_sm = launch_prep(p, kern, kAtCtaThreads, 0);
    const int sms = p->sms;
    const int64_t blocks = std::min<int64_t>(n_steps, static_cast<int64_t>(sms) * std::max(per_sm, 1));
    kern<<<static_cast<unsigned>(blocks), kAtCtaThreads, 0, s>>>(
        K, p->at_krow.as<int32_t>(), p->at_rows.as<int64_t>(), p->at_pos.as<PosT>(), n_steps, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

#ifndef FEA_PATCH_STAGES
#define FEA_PATCH_STAGES 4
#endif
constexpr int kTicketRing = 1024;
template <int D>
void run_atomic_patch(fea_plan* p, const double* K, double* values, cudaStream_t s) {
    constexpr int NPE = 8, P = kPatchElems, STAGES = FEA_PATCH_STAGES;
    constexpr int SLOT = D * NPE * D * NPE * 8 + NPE * NPE * 2;
    const int acc_doubles = ((p->pk_max_pairs + 1) * D * D + 1) & ~1;  // + spare pair; 16-byte aligned stages
    const size_t smem = static_cast<size_t>(acc_doubles) * 8 + STAGES * SLOT +
                        static_cast<size_t>(P * NPE) * 12 + static_cast<size_t>(P * NPE * NPE) * 2 + STAGES * 8 + 32;
    FEA_REQUIRE(smem <= 227 * 1024, FEA_ERR_INVALID, "patch accumulator too large");
    auto kern = k_atomic_patch<D, NPE, P, STAGES>;
    const int per_sm = launch_prep(p, kern, kPatchWarps * 32, smem);
    const int64_t blocks = std::min<int64_t>(p->pk_n, static_cast<int64_t>(p->sms) * std::max(per_sm, 1));
    if (blocks == 0) return;
    // one ticket counter per launch, from a ring (assemblies of one plan on several streams,
    // or several launches captured in one graph, must not share a live counter)
    // (long runs only: on cfg2, 44 patches per CTA, tickets measured 0.463 vs 0.444 ms - CTAs
    // that start together then flush the rows their neighbouring patches share at the same time)
    unsigned long long* ticket = nullptr;
    if (!p->kn.patch_static && (p->kn.patch_tickets || p->pk_n >= 256 * blocks)) {
        if (!p->pk_ticket.p) p->pk_ticket.alloc(kTicketRing * 8);
        ticket = p->pk_ticket.as<unsigned long long>() + (p->pk_ticket_next++ % kTicketRing);
        FEA_CK(cudaMemsetAsync(ticket, 0, 8, s));
    }
    kern<<<static_cast<unsigned>(blocks), kPatchWarps * 32, smem, s>>>(
        K, p->pk_hdr.as<int4>(), p->pk_krow.as<int32_t>(), p->pk_cidx.as<uint16_t>(), p->pk_rows.as<int64_t>(),
        p->pk_rowpair.as<int32_t>(), p->pk_pairs.as<uint16_t>(), p->pk_n, acc_doubles, ticket, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

void run_atomic_strip(fea_plan* p, const double* K, double* values, cudaStream_t s) {
    constexpr int STAGES = FEA_STRIP_STAGES;
    const size_t smem = static_cast<size_t>(STAGES) * (kStripElems * 128 + p->sk_stride + p->sk_sh_stride) + STAGES * 8 + 64;
    auto kern = k_atomic_strip<STAGES>;
    const int per_sm = launch_prep(p, kern, kStripThreads, smem);
    const int64_t blocks = std::min<int64_t>(p->sk_n, static_cast<int64_t>(p->sms) * std::max(per_sm, 1));
    if (blocks == 0) return;
    unsigned long long* ticket = nullptr;
    // grid stride by default: a strip takes ~2 us, so tickets for all CTAs would be ~440 M
    // same-address atomics per second (cfg3: 1.45 ms with tickets, 0.64 ms without)
    if (!p->kn.patch_static && p->kn.patch_tickets) {
        if (!p->pk_ticket.p) p->pk_ticket.alloc(kTicketRing * 8);
        ticket = p->pk_ticket.as<unsigned long long>() + (p->pk_ticket_next++ % kTicketRing);
        FEA_CK(cudaMemsetAsync(ticket, 0, 8, s));
    }
    kern<<<static_cast<unsigned>(blocks), kStripThreads, smem, s>>>(
        K, p->sk_meta.as<unsigned char>(), p->sk_shape.as<unsigned char>(), p->sk_k0.as<int4>(),
        p->sk_krow.as<int32_t>(), p->sk_n, p->sk_stride, p->sk_off_pos, p->sk_sh_stride, p->sk_off_prow,
        p->sk_off_ent, ticket, values);
    FEA_CK(cudaGetLastError());
    p->last_launches += 1;
}

template <class PosT>
bool atomic_staged(fea_plan* p, const double* K, double* values, cudaStream_t s) {
    if (p->sk_n > 0 && (reinterpret_cast<uintptr_t>(K) & 15u) == 0) {  // strip pre-reduction (npe 4, d 1)
        run_atomic_strip(p, K, values, s);
        return true;
    }
    if (p->pk_n > 0 && (reinterpret_cast<uintptr_t>(K) & 15u) == 0) {  // patch pre-reduction
        switch (p->d) {
            case 1: run_atomic_patch<1>(p, K, values, s); return true;
            case 2: run_atomic_patch<2>(p, K, values, s); return true;
            case 3: run_atomic_patch<3>(p, K, values, s); return true;
            default: break;
        }
    }
    if (!p->at_krow.p) return false;
    if ((reinterpret_cast<uintptr_t>(K) & 7u) == 0) {  // k_atomic_direct
        if (p->d == 3 && p->npe == 27) { run_atomic_cta<3, 27, PosT>(p, K, values, s); return true; }
        if (p->d == 1 && p->npe == 27) { run_atomic_cta<1, 27, PosT>(p, K, values, s); return true; }
    }
    if ((reinterpret_cast<uintptr_t>(K) & 15u) != 0) return false;
    switch (p->d * 16 + p->npe) {
        case 1 * 16 + 4: run_atomic_staged<1, 4, PosT>(p, K, values, s); return true;
        case 2 * 16 + 4: run_atomic_staged<2, 4, PosT>(p, K, values, s); return true;
        case 3 * 16 + 4: run_atomic_staged<3, 4, PosT>(p, K, values, s); return true;
        case 1 * 16 + 8: run_atomic_staged<1, 8, PosT>(p, K, values, s); return true;
        case 2 * 16 + 8: run_atomic_staged<2, 8, PosT>(p, K, values, s); return true;
        case 3 * 16 + 8: run_atomic_staged<3, 8, PosT>(p, K, values, s); return true;
        default: return false;
    }
}

}  // namespace
}  // namespace feagpu
