// Scan and radix sort of the symbolic phase (see prims.cuh).
#include "prims.cuh"

#include "internal.cuh"

namespace feagpu {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T warp_inclusive(T x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Exclusive prefix of `x` over the CTA (kScanThreads threads); *total = CTA sum.
template <class T>
__device__ __forceinline__ T block_exclusive(T x, T* total) {
    __shared__ T warp_tot[kScanThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T inc = warp_inclusive(x, lane);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    T before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
        const T t = warp_tot[w];
        if (w < warp) before += t;
        all += t;
    }
    *total = all;
    return before + inc - x;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* __restrict__ in, int64_t n,
                                                            T* __restrict__ sums) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
    T acc = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + j * kScanThreads + threadIdx.x;
        if (i < n) acc += in[i];
    }
    T total;
    block_exclusive(acc, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// in and out may alias: a thread holds its items in registers before it writes them.
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* in, T* out, int64_t n,
                                                            const T* __restrict__ tile_off) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile +
                         static_cast<int64_t>(threadIdx.x) * kScanItems;
    T v[kScanItems];
    T acc = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = base + j < n ? in[base + j] : T(0);
        acc += v[j];
    }
    T total;
    T run = block_exclusive(acc, &total) + (tile_off != nullptr ? tile_off[blockIdx.x] : T(0));
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < n) out[base + j] = run;
        run += v[j];
    }
}

template <class T>
void exclusive_sum_t(const T* in, T* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        k_tile_scan<T><<<1, kScanThreads, 0, s>>>(in, out, n, nullptr);
        FEA_CK(cudaGetLastError());
        return;
    }
    DevBuf sums;
    sums.alloc(static_cast<size_t>(tiles) * sizeof(T));
    k_tile_sums<T><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, sums.as<T>());
    FEA_CK(cudaGetLastError());
    exclusive_sum_t<T>(sums.as<T>(), sums.as<T>(), tiles, s);
    k_tile_scan<T><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, out, n, sums.as<T>());
    FEA_CK(cudaGetLastError());
    FEA_CK(cudaStreamSynchronize(s));  // `sums` is released on return
}

// ---- radix sort ----
constexpr int kRsWarps = 8;        // warps per CTA
constexpr int kRsChunk = 2048;     // consecutive items per warp
constexpr int kRsDigits = 256;

__global__ void __launch_bounds__(kRsWarps * 32) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n,
                                                              int shift, uint32_t mask, int64_t W,
                                                              uint32_t* __restrict__ table) {
    __shared__ uint32_t h[kRsWarps][kRsDigits];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kRsWarps + warp;
    if (w >= W) return;
    for (int dgt = lane; dgt < kRsDigits; dgt += 32) h[warp][dgt] = 0;
    __syncwarp();
    const int64_t i0 = w * kRsChunk, i1 = i0 + kRsChunk < n ? i0 + kRsChunk : n;
    for (int64_t i = i0 + lane; i < i1; i += 32) atomicAdd(&h[warp][(keys[i] >> shift) & mask], 1u);
    __syncwarp();
    for (int dgt = lane; dgt < kRsDigits; dgt += 32) table[static_cast<int64_t>(dgt) * W + w] = h[warp][dgt];
}

__global__ void __launch_bounds__(kRsWarps * 32) k_radix_scatter(
    const uint32_t* __restrict__ keys, const int32_t* __restrict__ vals, int64_t n, int shift, uint32_t mask,
    int64_t W, const uint32_t* __restrict__ table, uint32_t* __restrict__ keys_out, int32_t* __restrict__ vals_out) {
    __shared__ uint32_t off[kRsWarps][kRsDigits];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kRsWarps + warp;
    if (w >= W) return;
    for (int dgt = lane; dgt < kRsDigits; dgt += 32) off[warp][dgt] = table[static_cast<int64_t>(dgt) * W + w];
    __syncwarp();
    const int64_t i0 = w * kRsChunk, i1 = i0 + kRsChunk < n ? i0 + kRsChunk : n;
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t b = i0; b < i1; b += 32) {
        const int64_t i = b + lane;
        const bool ok = i < i1;
        const uint32_t act = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const uint32_t key = keys[i];
            const int32_t val = vals[i];
            const uint32_t dgt = (key >> shift) & mask;
            const uint32_t peers = __match_any_sync(act, dgt);
            const uint32_t rank = __popc(peers & lt);
            const uint32_t base = off[warp][dgt];
            __syncwarp(act);
            if (rank == 0) off[warp][dgt] = base + __popc(peers);
            __syncwarp(act);
            keys_out[base + rank] = key;
            vals_out[base + rank] = val;
        }
    }
}

}  // namespace

void exclusive_sum(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    exclusive_sum_t<int64_t>(in, out, n, s);
}
void exclusive_sum(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s) {
    exclusive_sum_t<uint32_t>(in, out, n, s);
}

void radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
                      int32_t* vals_out, int64_t n, int begin_bit, int end_bit, cudaStream_t s) {
    if (n <= 0) return;
    FEA_REQUIRE(n < (int64_t{1} << 31), FEA_ERR_INVALID, "radix sort of more than 2^31 items");
    int passes = (end_bit - begin_bit + 7) / 8;
    if (passes < 1) passes = 1;  // zero key bits: a stable copy
    const int64_t W = (n + kRsChunk - 1) / kRsChunk;
    const unsigned blocks = static_cast<unsigned>((W + kRsWarps - 1) / kRsWarps);
    DevBuf table, tk, tv;
    table.alloc(static_cast<size_t>(W) * kRsDigits * 4);
    if (passes > 1) {
        tk.alloc(static_cast<size_t>(n) * 4);
        tv.alloc(static_cast<size_t>(n) * 4);
    }
    const uint32_t* ksrc = keys_in;
    const int32_t* vsrc = vals_in;
    for (int ps = 0; ps < passes; ++ps) {
        const int shift = begin_bit + 8 * ps;
        const int nb = end_bit - shift < 8 ? (end_bit - shift > 0 ? end_bit - shift : 0) : 8;
        const uint32_t mask = (1u << nb) - 1u;
        // the last pass lands in keys_out / vals_out; earlier ones alternate with the temporaries
        const bool to_out = ((passes - 1 - ps) & 1) == 0;
        uint32_t* kdst = to_out ? keys_out : tk.as<uint32_t>();
        int32_t* vdst = to_out ? vals_out : tv.as<int32_t>();
        k_radix_hist<<<blocks, kRsWarps * 32, 0, s>>>(ksrc, n, shift, mask, W, table.as<uint32_t>());
        FEA_CK(cudaGetLastError());
        exclusive_sum(table.as<uint32_t>(), table.as<uint32_t>(), W * kRsDigits, s);
        k_radix_scatter<<<blocks, kRsWarps * 32, 0, s>>>(ksrc, vsrc, n, shift, mask, W, table.as<uint32_t>(),
                                                         kdst, vdst);
        FEA_CK(cudaGetLastError());
        ksrc = kdst;
        vsrc = vdst;
    }
    FEA_CK(cudaStreamSynchronize(s));  // temporaries are released on return
}

}  // namespace feagpu
