// Numeric phase of the B200 FE-assembly library (north-star subsystem 3): the scatter-add
// G(D(r), D(c)) += K_e(r, c) of scatter_element (assembly.hpp:77-92) for all elements, with
// three conflict strategies (kernels in kernels.cuh, instantiated per position width in
// gather_u8.cu / gather_u16.cu):
//
//  FEA_DET_SORTED  owner-computes segmented reduction (k_gather_cn / k_gather_node /
//      k_gather_stream). A lane group owns a node's d rows (a contiguous block of values); it
//      streams the node's incident element-matrix row blocks K[e][a*d .. a*d+d-1][:] in
//      ascending element id and folds them into a shared-memory copy of the block, then writes
//      the block once. Per slot: a left fold from the slot's start value in ascending element
//      order — bit-identical to assemble_sequential (assembly.hpp:112-118). K read once, values
//      written once, no atomics.
//  FEA_DET_COLOUR  the same reduction over incidences ordered by (colour, element): per slot
//      the colour order of assemble_coloured_vectorized (assembly.hpp:175-195), bit-identical;
//      FEA_COLOUR_PASSES runs it literally, one k_scatter<plain> launch per colour.
//  FEA_ATOMIC      k_scatter<atomic>: element owner, one fp64 atomicAdd (RED.E.ADD.F64) per
//      entry, elements in a locality order (assemble_atomic, assembly.hpp:121-126).
#include <cstring>
#include <exception>
#include <thread>
#include <unordered_map>

#include <chrono>

#include "kernels.cuh"

namespace feagpu {

void build_atomic_maps(fea_plan* p, cudaStream_t s);
void build_patches(fea_plan* p, cudaStream_t s);
void build_strips(fea_plan* p, cudaStream_t s);

// --- lattice-like item sequences and their tiled visit order ----------------------------------
// Items (the patches of k_atomic_patch) in visit order. On a structured
// mesh in lexicographic order item q shares nodes with q + 1, q + s1 +- 1, q + s1, q + s2 +- s1 +- 1,
// ...: the strides are read off an interior item's later neighbours and checked on 257 samples
// (no geometry in the plan). later(q, out) fills the sorted distinct offsets nb - q of the items
// nb > q that share a node with q.
template <class Later>
bool detect_lattice(int64_t n, Later&& later, int64_t* s1_out, int64_t* s2_out) {
    std::vector<int64_t> offs;
    int64_t s1 = 0, s2 = 0;
    for (int smp = 0; smp < 64 && s1 == 0 && n > 0; ++smp) {  // an interior item: 13 later neighbours
        later((n / 2 + smp * (std::max<int64_t>(n / 67, 1) | 1)) % n, offs);
        if (offs.size() == 13 && offs[0] == 1 && offs[1] + 1 == offs[2] && offs[2] + 1 == offs[3]) {
            s1 = offs[2];
            s2 = offs[8];
        }
    }
    bool lattice = s1 > 1 && s2 > s1 && s2 % s1 == 0 && n >= 2 * s2;
    if (lattice) {
        const int64_t want[13] = {1, s1 - 1, s1, s1 + 1, s2 - s1 - 1, s2 - s1, s2 - s1 + 1, s2 - 1, s2, s2 + 1,
                                  s2 + s1 - 1, s2 + s1, s2 + s1 + 1};
        for (int smp = 0; smp < 257 && lattice; ++smp) {
            later((n - 1) * smp / 256, offs);
            for (int64_t o : offs) lattice = lattice && std::find(want, want + 13, o) != want + 13;
        }
    }
    *s1_out = s1;
    *s2_out = s2;
    return lattice;
}

// Sequence positions re-ordered into tiles of T x T columns visited plane after plane: the items
// of the next plane follow T * T positions later instead of s2 (a whole plane, which outgrows
// the L2 on large meshes, so every values row shared between two planes was fetched twice).
std::vector<int32_t> tiled_sequence(int64_t n, int64_t s1, int64_t s2, int T) {
    const int64_t nx = s1, ny = s2 / s1, tiles_x = (nx + T - 1) / T;
    std::vector<int32_t> seq(static_cast<size_t>(n));
    for (int64_t q = 0; q < n; ++q) seq[q] = static_cast<int32_t>(q);
    if (tiles_x * ((ny + T - 1) / T) >= (int64_t{1} << 23) || n / s2 >= (int64_t{1} << 20) || T * T >= (1 << 20))
        return seq;
    std::vector<std::pair<uint64_t, int32_t>> key(static_cast<size_t>(n));
    for (int64_t q = 0; q < n; ++q) {
        const int64_t x = q % s1, y = (q % s2) / s1, z = q / s2;
        const uint64_t tile = static_cast<uint64_t>((y / T) * tiles_x + x / T);
        key[q] = {(tile << 40) | (static_cast<uint64_t>(z) << 20) | static_cast<uint64_t>((y % T) * T + x % T),
                  static_cast<int32_t>(q)};
    }
    std::sort(key.begin(), key.end());
    for (int64_t q = 0; q < n; ++q) seq[q] = key[q].second;
    return seq;
}

void ensure_element_maps(fea_plan* p, cudaStream_t s) {
    if (p->posE.p && p->order.p) return;
    const int64_t n = p->E * p->npe * p->npe;
    p->posE.alloc(n * p->pos_bytes);
    FEA_CK(cudaMemsetAsync(p->posE.p, 0xff, p->posE.bytes, s));
    DevBuf k2l;
    const int32_t* k2l_ptr = nullptr;
    if (p->partitioned && !p->k_compact) {
        k2l.alloc(p->E_in * 4);
        if (p->E > 0)
            k_k2l<<<grid_for(p->E, 256), 256, 0, s>>>(p->elem_krow.as<int32_t>(), p->E,
                                                      k2l.as<int32_t>());
        k2l_ptr = k2l.as<int32_t>();
    }
    if (p->n_adj > 0) {
        if (p->pos_bytes == 1)
            k_pos_elem<uint8_t><<<grid_for(p->n_adj * p->npe, 256), 256, 0, s>>>(
                p->adj.as<int32_t>(), p->posA.as<uint8_t>(), p->n_adj, p->npe, p->pstride, k2l_ptr,
                p->posE.as<uint8_t>());
        else
            k_pos_elem<uint16_t><<<grid_for(p->n_adj * p->npe, 256), 256, 0, s>>>(
                p->adj.as<int32_t>(), p->posA.as<uint16_t>(), p->n_adj, p->npe, p->pstride, k2l_ptr,
                p->posE.as<uint16_t>());
    }
    FEA_CK(cudaGetLastError());
    // Atomic-route element order: keep the caller's order when consecutive
    // elements already share nodes (>= half the pairs), else visit elements
    // sorted by their lowest node id so concurrently resident CTAs hit the
    // same rows and the reductions stay in L2.
    p->order.alloc(p->E * 4);
    if (p->E > 0) {
        DevBuf keys, vals, keys2, cnt;
        keys.alloc(p->E * 4);
        vals.alloc(p->E * 4);
        keys2.alloc(p->E * 4);
        cnt.alloc(8);
        FEA_CK(cudaMemsetAsync(cnt.p, 0, 8, s));
        k_locality<<<grid_for(p->E, 256), 256, 0, s>>>(p->conn_k.as<int32_t>(),
                                                       p->elem_krow.as<int32_t>(), p->E, p->npe,
                                                       cnt.as<unsigned long long>(),
                                                       keys.as<uint32_t>(), vals.as<int32_t>());
        FEA_CK(cudaGetLastError());
        unsigned long long shared = 0;
        FEA_CK(cudaMemcpyAsync(&shared, cnt.p, 8, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        if (2 * static_cast<int64_t>(shared) >= p->E - 1) {
            k_iota32<<<grid_for(p->E, 256), 256, 0, s>>>(p->order.as<int32_t>(), p->E);
        } else {
            radix_sort_pairs(keys.as<uint32_t>(), keys2.as<uint32_t>(), vals.as<int32_t>(),
                             p->order.as<int32_t>(), p->E, 0, 32, s);
        }
        FEA_CK(cudaGetLastError());
        FEA_CK(cudaStreamSynchronize(s));
    }
    build_atomic_maps(p, s);
    build_patches(p, s);
    build_strips(p, s);
}

// --- patch tables on the device -----------------------------------------------------------------
// One warp per patch (P = 8 element slots of npe = 8 nodes): the patch's owned row nodes in order
// of first appearance, and its distinct (row, position) pairs, keys row << 8 | position, sorted
// and made unique - a warp bitonic sort in shared memory like the symbolic phase's
// k_node_pattern. FILL = false counts rows and pairs per patch; after the two
// exclusive scans FILL = true writes the header, the row words, the row pair ranges, the pair
// list, the K row of every element slot and the pair index of every (slot, a, b).
constexpr int kPtWarps = 4;
__device__ __forceinline__ void patch_bitonic(int32_t* s, int n, int lane) {  // n: power of two
    for (int k = 2; k <= n; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < n; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int32_t a = s[i], b = s[ixj];
                    if ((a > b) == ((i & k) == 0)) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncwarp();
        }
}
// compact the distinct values of sorted s[0..n) (INT32_MAX = none) to its front; returns the count
__device__ __forceinline__ int patch_unique(int32_t* s, int n, int lane) {
    int total = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const int32_t x = s[i];
        const bool uniq = x != INT32_MAX && (i == 0 || x != s[i - 1]);
        const unsigned bal = __ballot_sync(0xffffffffu, uniq);
        __syncwarp();  // every lane has read s[i] and s[i - 1] of this step
        if (uniq) s[total + __popc(bal & ((1u << lane) - 1u))] = x;  // total + rank <= i: no later step reads it
        total += __popc(bal);
        __syncwarp();
    }
    return total;
}
__device__ __forceinline__ int patch_find(const int32_t* s, int n, int32_t x) {  // x is present
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
template <bool FILL>
__global__ void __launch_bounds__(kPtWarps * 32)
    k_patch_tables(const int32_t* __restrict__ members, int64_t n_patch, const int32_t* __restrict__ elem_krow,
                   const int32_t* __restrict__ conn_k, const uint8_t* __restrict__ posE,
                   const int64_t* __restrict__ nptr, int64_t node_begin, int64_t n_own, int d,
                   int64_t* __restrict__ n_rows_out, int64_t* __restrict__ n_pairs_out,
                   const int64_t* __restrict__ row_off, const int64_t* __restrict__ pair_off, int max_pairs,
                   int4* __restrict__ hdr, int32_t* __restrict__ pk_krow, uint16_t* __restrict__ pk_cidx,
                   int64_t* __restrict__ pk_rows, int32_t* __restrict__ pk_rowpair, uint16_t* __restrict__ pk_pairs) {
    constexpr int P = kPatchElems, NPE = 8, NN = 64;
    __shared__ int32_t s_node[kPtWarps][P * NPE];
    __shared__ int32_t s_cand[kPtWarps][P * NPE];
    __shared__ int32_t s_key[kPtWarps][P * NN];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t* rows = s_node[w];
    int32_t* cand = s_cand[w];
    int32_t* keys = s_key[w];
    for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < n_patch;
         q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        // the patch's (slot, a) nodes: 64 entries, two per lane
        int32_t le[2], nd[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int x = lane + 32 * h, k = x / NPE, a = x - k * NPE;
            le[h] = members[q * P + k];
            nd[h] = INT32_MAX;
            if (le[h] >= 0) {
                const int32_t v = conn_k[static_cast<int64_t>(elem_krow[le[h]]) * NPE + a];
                if (v >= node_begin && v - node_begin < n_own) nd[h] = v;
            }
            cand[x] = nd[h];
        }
        __syncwarp();
        // rows in order of first appearance over (slot, a) - the order the flush walks them in
        // (sorted by node id measured 2 % slower on cfg2 and config 5): an entry is a row's first
        // when no earlier entry names its node; its row index is the number of firsts before it
        int fx[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int x = lane + 32 * h;
            fx[h] = x;
            if (nd[h] != INT32_MAX)
                for (int y = 0; y < x; ++y)
                    if (cand[y] == nd[h]) {
                        fx[h] = y;
                        break;
                    }
        }
        const unsigned f0 = __ballot_sync(0xffffffffu, nd[0] != INT32_MAX && fx[0] == lane);
        const unsigned f1 = __ballot_sync(0xffffffffu, nd[1] != INT32_MAX && fx[1] == lane + 32);
        auto rank_of = [&](int y) {
            return y < 32 ? __popc(f0 & ((1u << y) - 1u)) : __popc(f0) + __popc(f1 & ((1u << (y - 32)) - 1u));
        };
        const int n_rows = __popc(f0) + __popc(f1);
        int r[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            r[h] = nd[h] != INT32_MAX ? rank_of(fx[h]) : -1;
            if (r[h] >= 0 && fx[h] == lane + 32 * h) rows[r[h]] = nd[h];
        }
        // pair keys: row << 8 | position of every entry (slot, a, b) with an owned row node
        for (int x = lane; x < P * NN; x += 32) keys[x] = INT32_MAX;
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (r[h] >= 0) {
                const int x = lane + 32 * h;
                const uint2 pz = *reinterpret_cast<const uint2*>(posE + static_cast<int64_t>(le[h]) * NN + (x % NPE) * NPE);
#pragma unroll
                for (int b = 0; b < NPE; ++b)
                    keys[x * NPE + b] = (r[h] << 8) | static_cast<int>(((b < 4 ? pz.x : pz.y) >> (8 * (b & 3))) & 0xffu);
            }
        }
        __syncwarp();
        patch_bitonic(keys, P * NN, lane);
        const int n_pairs = patch_unique(keys, P * NN, lane);
        if (!FILL) {
            if (lane == 0) {
                n_rows_out[q] = n_rows;
                n_pairs_out[q] = n_pairs;
            }
        } else {
            const int64_t ro = row_off[q], po = pair_off[q];
            int n_el = 0;
            for (int k = 0; k < P; ++k) n_el += members[q * P + k] >= 0;
            if (lane == 0)
                hdr[q] = make_int4(0, static_cast<int>(po), static_cast<int>(ro), n_el | (n_rows << 8) | (n_pairs << 16));
            if (lane < P) {
                const int32_t e = members[q * P + lane];
                pk_krow[q * P + lane] = e >= 0 ? elem_krow[e] : -1;
            }
            for (int i = lane; i < n_rows; i += 32) {
                const int64_t vo = rows[i] - node_begin, c0 = nptr[vo];
                pk_rows[ro + i] = ((static_cast<int64_t>(d) * d * c0) << 20) | (static_cast<int64_t>(d) * (nptr[vo + 1] - c0));
                // pairs are sorted by row: the row's range is [first key >= i << 8, first key >= (i + 1) << 8)
                int lo = 0, hi = n_pairs;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (keys[mid] < (i << 8)) lo = mid + 1;
                    else hi = mid;
                }
                int lo2 = lo, hi2 = n_pairs;
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2) >> 1;
                    if (keys[mid] < ((i + 1) << 8)) lo2 = mid + 1;
                    else hi2 = mid;
                }
                pk_rowpair[ro + i] = lo | ((lo2 - lo) << 16);
            }
            for (int i = lane; i < n_pairs; i += 32) pk_pairs[po + i] = static_cast<uint16_t>(keys[i]);
            // pair index of every entry; a row node outside the owned range -> the spare pair
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (le[h] < 0) continue;
                const int x = lane + 32 * h;
                uint16_t* out = pk_cidx + (q * P + x / NPE) * NN + (x % NPE) * NPE;
                const uint2 pz = *reinterpret_cast<const uint2*>(posE + static_cast<int64_t>(le[h]) * NN + (x % NPE) * NPE);
#pragma unroll
                for (int b = 0; b < NPE; ++b) {
                    const int pos = static_cast<int>(((b < 4 ? pz.x : pz.y) >> (8 * (b & 3))) & 0xffu);
                    const int idx = r[h] >= 0 ? patch_find(keys, n_pairs, (r[h] << 8) | pos) : max_pairs;
                    FEA_DCHECK(r[h] < 0 || (idx < n_pairs && keys[idx] == ((r[h] << 8) | pos)));
                    out[b] = static_cast<uint16_t>(idx);
                }
            }
        }
        __syncwarp();
    }
}

__global__ void k_max2_i64(const int64_t* __restrict__ a, const int64_t* __restrict__ b, int64_t n,
                           unsigned long long* out) {  // out[0] = max a, out[1] = max b
    unsigned long long ma = 0, mb = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        ma = max(ma, static_cast<unsigned long long>(a[i]));
        mb = max(mb, static_cast<unsigned long long>(b[i]));
    }
    for (int o = 16; o > 0; o >>= 1) {
        ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, ma);
        atomicMax(out + 1, mb);
    }
}

// --- patches as node stars, found on the device ----------------------------------------------------
// A 2 x 2 x 2 block of hex8 elements is the star of its centre node. On a plan that owns every
// row the patches can therefore be found without the host's sequential sweep: candidates are the
// nodes with exactly P incident elements, the chosen centres are the lexicographically first
// maximal independent set of candidates in the node graph (two nodes that share an element are
// neighbours - the pattern's rows - so chosen stars are disjoint), found by rounds: an undecided
// candidate is chosen once every lower-numbered neighbouring candidate is out, and is out once one
// of them is chosen. On a structured mesh in lexicographic numbering that is the host sweep's
// tiling (centres at odd coordinates) in ~n rounds. The route is taken only if the stars cover
// every element (even element counts per direction); anything else keeps the host sweep.
__global__ void k_star_init(const int64_t* __restrict__ adj_ptr, int64_t n, int P, uint8_t* __restrict__ state) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        state[v] = adj_ptr[v + 1] - adj_ptr[v] == P ? 0 : 2;  // 0 undecided, 1 chosen, 2 out
}
__global__ void k_star_round(const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol, int64_t n,
                             volatile uint8_t* state, unsigned long long* __restrict__ undecided) {
    unsigned long long mine = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (state[v] != 0) continue;
        bool wait = false, kill = false;
        for (int64_t j = nptr[v]; j < nptr[v + 1]; ++j) {
            const int32_t u = ncol[j];
            if (u >= v) break;  // ascending: only lower-numbered neighbours decide
            const uint8_t su = state[u];  // a stale "undecided" only delays the decision by a round
            kill = kill || su == 1;
            wait = wait || su == 0;
        }
        if (kill) state[v] = 2;
        else if (!wait) state[v] = 1;
        else ++mine;
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(undecided, mine);
}
__global__ void k_star_flags(const uint8_t* __restrict__ state, int64_t n, int64_t* __restrict__ flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x)
        flag[v] = v < n && state[v] == 1;
}
// members of every chosen star (its incident elements in adjacency order) and the patch of each
__global__ void k_star_members(const uint8_t* __restrict__ state, const int64_t* __restrict__ idx, int64_t n,
                               const int64_t* __restrict__ adj_ptr, const int32_t* __restrict__ adj, int npe, int P,
                               int32_t* __restrict__ members, int32_t* __restrict__ patch_of) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (state[v] != 1) continue;
        const int64_t q = idx[v], b0 = adj_ptr[v];
        // slot of an element = where the centre sits in it: for the usual hex8 local numbering the
        // order below walks the block's elements lexicographically, whatever their ids are (the
        // host sweep's order; by ascending id cfg2's permuted elements measured 2.5 % slower)
        const int rank[8] = {7, 6, 4, 5, 3, 2, 0, 1};
        int32_t slot[8];
        for (int k = 0; k < 8; ++k) slot[k] = -1;
        for (int k = 0; k < P; ++k) {
            const int32_t entry = adj[b0 + k];
            const int a = entry % npe;
            if (a < 8 && slot[rank[a]] < 0) slot[rank[a]] = entry / npe;  // the plan owns every row: K row = element
        }
        for (int k = 0; k < P; ++k) {  // two elements with the centre at the same local node: first free slot
            const int32_t entry = adj[b0 + k];
            const int a = entry % npe;
            if (a < 8 && slot[rank[a]] == entry / npe) continue;
            for (int f = 0; f < P; ++f)
                if (slot[f] < 0) {
                    slot[f] = entry / npe;
                    break;
                }
        }
        for (int k = 0; k < P; ++k) {
            members[q * P + k] = slot[k];
            patch_of[slot[k]] = static_cast<int32_t>(q);
        }
    }
}
// offsets nb - q of the patches nb > q that share a node with sampled patch q (0: none), 64 x 8 slots
__global__ void k_patch_later(const int64_t* __restrict__ samples, const int32_t* __restrict__ members,
                              const int32_t* __restrict__ conn_k, const int64_t* __restrict__ adj_ptr,
                              const int32_t* __restrict__ adj, const int32_t* __restrict__ patch_of, int npe, int P,
                              int64_t* __restrict__ out) {
    const int64_t q = samples[blockIdx.x];
    const int t = threadIdx.x, k = t / npe, a = t - k * npe;  // blockDim = P * npe
    int64_t* o = out + (static_cast<int64_t>(blockIdx.x) * blockDim.x + t) * 8;
    for (int j = 0; j < 8; ++j) o[j] = 0;
    const int32_t le = members[q * P + k];
    if (le < 0) return;
    const int64_t v = conn_k[static_cast<int64_t>(le) * npe + a];
    const int64_t b0 = adj_ptr[v];
    const int n = static_cast<int>(min(adj_ptr[v + 1] - b0, static_cast<int64_t>(8)));
    for (int j = 0; j < n; ++j) {
        const int64_t nb = patch_of[adj[b0 + j] / npe];
        o[j] = nb > q ? nb - q : 0;
    }
}
// tiled_sequence on the device: the key (tile, z, position in the tile) of item vals[i], one part
// per stable radix pass (least significant part first)
__global__ void k_tile_key(const int32_t* __restrict__ vals, int64_t n, int64_t s1, int64_t s2, int T, int part,
                           uint32_t* __restrict__ keys) {
    const int64_t tiles_x = (s1 + T - 1) / T;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = vals ? vals[i] : i;
        const int64_t x = q % s1, y = (q % s2) / s1, z = q / s2;
        keys[i] = static_cast<uint32_t>(part == 0 ? (y % T) * T + x % T : part == 1 ? z : (y / T) * tiles_x + x / T);
    }
}
__global__ void k_permute_members(const int32_t* __restrict__ seq, const int32_t* __restrict__ in, int64_t n, int P,
                                  int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * P; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[static_cast<int64_t>(seq[i / P]) * P + i % P];
}

// Patches of k_atomic_patch (npe = 8, d <= 3, byte positions, no repeated nodes): greedy growth
// from the atomic visit order — the first unassigned element, then repeatedly the unassigned
// element sharing the most nodes with the patch (ties: earlier in the visit order) — up to
// kPatchElems elements; on structured hex8 meshes this tiles 2 x 2 x 2 blocks. Per patch the
// distinct (owned row node, column node) pairs, sorted by (row, position), and per element the
// pair index of each (a, b). Once per plan, on the first atomic assembly. Where the node stars
// tile the mesh the patches are found on the device (star_patches); otherwise the greedy growth
// (a sequential sweep) and the lattice order run on the host. The tables are built on the device
// either way (k_patch_tables; 12 s of a 16 s first call on config 5 when one host thread built them).
// Device route of build_patches (see k_star_init). false: the stars do not tile the mesh.
bool star_patches(fea_plan* p, DevBuf& d_mem, int64_t* n_patch_out, cudaStream_t s) {
    constexpr int P = kPatchElems;
    const int64_t n = p->n_own, E = p->E;
    if (p->partitioned || n == 0 || p->n_adj != E * p->npe || std::getenv("FEA_PATCH_HOST_SWEEP")) return false;
    const bool trace = std::getenv("FEA_PLAN_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "star trace:  %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    DevBuf state, cnt, flag, idx, patch_of, bad;
    state.alloc(n);
    cnt.alloc(8);
    k_star_init<<<grid_for(n, 256), 256, 0, s>>>(p->adj_ptr.as<int64_t>(), n, P, state.as<uint8_t>());
    FEA_CK(cudaGetLastError());
    for (int round = 0;; round += 8) {  // 8 rounds per look at the counter
        if (round >= 4096) return false;  // a long dependency chain (a thin bar of elements): host sweep
        unsigned long long left = 0;
        for (int r = 0; r < 8; ++r) {
            FEA_CK(cudaMemsetAsync(cnt.p, 0, 8, s));
            k_star_round<<<grid_for(n, 256), 256, 0, s>>>(p->nptr.as<int64_t>(), p->ncol.as<int32_t>(), n,
                                                         state.as<uint8_t>(), cnt.as<unsigned long long>());
        }
        FEA_CK(cudaGetLastError());
        FEA_CK(cudaMemcpyAsync(&left, cnt.p, 8, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        if (left == 0) break;
    }
    mark("selection rounds");
    flag.alloc((n + 1) * 8);
    idx.alloc((n + 1) * 8);
    k_star_flags<<<grid_for(n + 1, 256), 256, 0, s>>>(state.as<uint8_t>(), n, flag.as<int64_t>());
    exclusive_sum(flag.as<int64_t>(), idx.as<int64_t>(), n + 1, s);
    int64_t n_patch = 0;
    FEA_CK(cudaMemcpyAsync(&n_patch, idx.as<int64_t>() + n, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    if (n_patch * P != E) return false;  // disjoint stars of P elements each: they cover the mesh iff the counts agree
    d_mem.alloc(static_cast<size_t>(n_patch) * P * 4);
    patch_of.alloc(static_cast<size_t>(E) * 4);
    k_star_members<<<grid_for(n, 256), 256, 0, s>>>(state.as<uint8_t>(), idx.as<int64_t>(), n, p->adj_ptr.as<int64_t>(),
                                                   p->adj.as<int32_t>(), p->npe, P, d_mem.as<int32_t>(),
                                                   patch_of.as<int32_t>());
    FEA_CK(cudaGetLastError());
    mark("members");
    // lattice order of the patch sequence (as in the host route): later neighbours of the sampled
    // patches from a small kernel, the tile permutation applied on the device
    if (!std::getenv("FEA_PATCH_NO_TILES")) {
        std::vector<int64_t> samples;
        for (int smp = 0; smp < 64; ++smp) samples.push_back((n_patch / 2 + smp * (std::max<int64_t>(n_patch / 67, 1) | 1)) % n_patch);
        for (int smp = 0; smp < 257; ++smp) samples.push_back((n_patch - 1) * smp / 256);
        const int threads = P * p->npe;
        DevBuf d_s, d_o;
        d_s.alloc(samples.size() * 8);
        d_o.alloc(samples.size() * threads * 8 * 8);
        FEA_CK(cudaMemcpyAsync(d_s.p, samples.data(), samples.size() * 8, cudaMemcpyHostToDevice, s));
        k_patch_later<<<static_cast<unsigned>(samples.size()), threads, 0, s>>>(
            d_s.as<int64_t>(), d_mem.as<int32_t>(), p->conn_k.as<int32_t>(), p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(),
            patch_of.as<int32_t>(), p->npe, P, d_o.as<int64_t>());
        FEA_CK(cudaGetLastError());
        std::vector<int64_t> h_o(samples.size() * threads * 8);
        FEA_CK(cudaMemcpyAsync(h_o.data(), d_o.p, h_o.size() * 8, cudaMemcpyDeviceToHost, s));
        FEA_CK(cudaStreamSynchronize(s));
        auto later = [&](int64_t q, std::vector<int64_t>& offs) {
            offs.clear();
            const size_t i = static_cast<size_t>(std::find(samples.begin(), samples.end(), q) - samples.begin());
            if (i == samples.size()) return;
            for (int t = 0; t < threads * 8; ++t)
                if (h_o[i * threads * 8 + t] > 0) offs.push_back(h_o[i * threads * 8 + t]);
            std::sort(offs.begin(), offs.end());
            offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
        };
        int64_t s1 = 0, s2 = 0;
        const bool lattice = detect_lattice(n_patch, later, &s1, &s2);
        mark("lattice detection");
        const int64_t plane_k = s2 * P * static_cast<int64_t>(p->m) * p->m * 8;
        if (std::getenv("FEA_PATCH_DEBUG"))
            std::fprintf(stderr, "patch lattice (stars): n_patch %lld s1 %lld s2 %lld lattice %d plane_k %lld\n",
                         (long long)n_patch, (long long)s1, (long long)s2, (int)lattice, (long long)plane_k);
        const char* tile_env = std::getenv("FEA_PATCH_TILE");
        if (lattice && (plane_k > (int64_t{64} << 20) || tile_env)) {
            // tiled_sequence(): three stable radix passes over the key parts instead of a host sort
            const int T = tile_env ? std::max(1, std::atoi(tile_env)) : 16;
            const int64_t tiles = ((s1 + T - 1) / T) * ((s2 / s1 + T - 1) / T), nz = (n_patch + s2 - 1) / s2;
            DevBuf d_seq, d_m2, k_in, k_out, v_a, v_b;
            d_m2.alloc(d_mem.bytes);
            k_in.alloc(n_patch * 4);
            k_out.alloc(n_patch * 4);
            v_a.alloc(n_patch * 4);
            v_b.alloc(n_patch * 4);
            k_iota32<<<grid_for(n_patch, 256), 256, 0, s>>>(v_a.as<int32_t>(), n_patch);
            const uint64_t span[3] = {static_cast<uint64_t>(T) * T, static_cast<uint64_t>(nz), static_cast<uint64_t>(tiles)};
            DevBuf* src = &v_a;
            DevBuf* dst = &v_b;
            for (int part = 0; part < 3; ++part) {
                k_tile_key<<<grid_for(n_patch, 256), 256, 0, s>>>(src->as<int32_t>(), n_patch, s1, s2, T, part,
                                                                 k_in.as<uint32_t>());
                int bits = 1;
                while (bits < 32 && (uint64_t{1} << bits) < span[part]) ++bits;
                radix_sort_pairs(k_in.as<uint32_t>(), k_out.as<uint32_t>(), src->as<int32_t>(), dst->as<int32_t>(), n_patch, 0,
                                 bits, s);
                std::swap(src, dst);
            }
            FEA_CK(cudaGetLastError());
            d_seq = std::move(*src);
            k_permute_members<<<grid_for(n_patch * P, 256), 256, 0, s>>>(d_seq.as<int32_t>(), d_mem.as<int32_t>(), n_patch, P,
                                                                        d_m2.as<int32_t>());
            FEA_CK(cudaGetLastError());
            FEA_CK(cudaStreamSynchronize(s));
            d_mem = std::move(d_m2);
        }
    } else if (std::getenv("FEA_PATCH_DEBUG")) {
        std::fprintf(stderr, "patch stars: n_patch %lld\n", (long long)n_patch);
    }
    mark("tile order");
    *n_patch_out = n_patch;
    return true;
}

void build_patches(fea_plan* p, cudaStream_t s) {
    if (p->npe != 8 || p->d > 3 || p->pos_bytes != 1 || p->dup_nodes || p->E == 0 || p->kn.atomic_no_patch ||
        p->kn.atomic_legacy || p->pk_n > 0)
        return;
    constexpr int NPE = 8, NN = 64, P = kPatchElems;
    const int64_t E = p->E;
    const bool trace = std::getenv("FEA_PLAN_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "patch trace: %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    DevBuf d_mem;
    int64_t n_patch = 0;
    const bool on_device = star_patches(p, d_mem, &n_patch, s);
    if (on_device) mark("star patches (device)");
    if (!on_device) {
    std::vector<int32_t> order(E), krow(E), conn(static_cast<size_t>(p->krows() * NPE));
    FEA_CK(cudaMemcpyAsync(order.data(), p->order.p, E * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(krow.data(), p->elem_krow.p, E * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(conn.data(), p->conn_k.p, conn.size() * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    auto node = [&](int64_t le, int a) { return conn[static_cast<size_t>(krow[le]) * NPE + a]; };
    int32_t max_node = 0;
    for (int64_t le = 0; le < E; ++le)
        for (int a = 0; a < NPE; ++a) max_node = std::max(max_node, node(le, a));
    const int64_t nn = static_cast<int64_t>(max_node) + 1;
    // node -> elements (local ids)
    std::vector<int64_t> aptr(nn + 1, 0);
    for (int64_t le = 0; le < E; ++le)
        for (int a = 0; a < NPE; ++a) ++aptr[node(le, a) + 1];
    for (int64_t v = 0; v < nn; ++v) aptr[v + 1] += aptr[v];
    std::vector<int32_t> aelem(static_cast<size_t>(aptr[nn]));
    {
        std::vector<int64_t> fill(aptr.begin(), aptr.end() - 1);
        for (int64_t le = 0; le < E; ++le)
            for (int a = 0; a < NPE; ++a) aelem[fill[node(le, a)]++] = static_cast<int32_t>(le);
    }
    std::vector<int32_t> vpos(E);
    for (int64_t i = 0; i < E; ++i) vpos[order[i]] = static_cast<int32_t>(i);
    mark("copies + node->element index");
    // greedy patches
    std::vector<char> assigned(E, 0);
    std::vector<int32_t> stamp(E, -1);
    std::vector<int16_t> cnt(E, 0);
    std::vector<int32_t> members;  // P per patch, -1 padded
    members.reserve(static_cast<size_t>(E / 4 + P));
    std::vector<int32_t> cand;
    int32_t pid = 0;
    for (int64_t i = 0; i < E; ++i) {
        const int32_t e0 = order[i];
        if (assigned[e0]) continue;
        cand.clear();
        int n_m = 0;
        auto add = [&](int32_t e) {
            assigned[e] = 1;
            members.push_back(e);
            ++n_m;
            for (int a = 0; a < NPE; ++a) {
                const int32_t v = node(e, a);
                for (int64_t k = aptr[v]; k < aptr[v + 1]; ++k) {
                    const int32_t g = aelem[k];
                    if (assigned[g]) continue;
                    if (stamp[g] != pid) {
                        stamp[g] = pid;
                        cnt[g] = 0;
                        cand.push_back(g);
                    }
                    ++cnt[g];
                }
            }
        };
        add(e0);
        while (n_m < P) {
            int32_t best = -1;
            for (int32_t g : cand)
                if (!assigned[g] && (best < 0 || cnt[g] > cnt[best] || (cnt[g] == cnt[best] && vpos[g] < vpos[best])))
                    best = g;
            if (best < 0) break;
            add(best);
        }
        for (; n_m < P; ++n_m) members.push_back(-1);
        ++pid;
    }
    n_patch = pid;
    mark("greedy growth");
    // Tiled visit order for lattice-like patch sequences (a structured mesh in lexicographic
    // order: patch q shares nodes with q + 1, q + s1 +- 1, q + s2 +- s1 +- 1). In sequence order
    // the patches of the next plane come s2 patches later (config 5: 16,384 patches = 0.6 GB of
    // K), so the values rows of every node plane between two patch planes are fetched and
    // written back twice. Visiting tiles of T x T patch columns plane after plane brings the next
    // plane's patches T * T tickets later. The strides are detected from the patch adjacency
    // (no geometry in the plan); any other sequence keeps its order. Any order is valid.
    if (n_patch > 0 && !std::getenv("FEA_PATCH_NO_TILES")) {
        std::vector<int32_t> patch_of(E, -1);
        for (int64_t q = 0; q < n_patch; ++q)
            for (int k = 0; k < P; ++k)
                if (members[q * P + k] >= 0) patch_of[members[q * P + k]] = static_cast<int32_t>(q);
        auto later = [&](int64_t q, std::vector<int64_t>& offs) {
            offs.clear();
            for (int k = 0; k < P; ++k) {
                const int32_t le = members[q * P + k];
                if (le < 0) continue;
                for (int a = 0; a < NPE; ++a) {
                    const int32_t v = node(le, a);
                    for (int64_t j = aptr[v]; j < aptr[v + 1]; ++j) {
                        const int64_t nb = patch_of[aelem[j]];
                        if (nb > q) offs.push_back(nb - q);
                    }
                }
            }
            std::sort(offs.begin(), offs.end());
            offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
        };
        int64_t s1 = 0, s2 = 0;
        const bool lattice = detect_lattice(n_patch, later, &s1, &s2);
        // only where a plane of patches outgrows the L2 (K bytes of one plane)
        const int64_t plane_k = s2 * P * static_cast<int64_t>(p->m) * p->m * 8;
        if (std::getenv("FEA_PATCH_DEBUG"))
            std::fprintf(stderr, "patch lattice: n_patch %lld s1 %lld s2 %lld lattice %d plane_k %lld\n",
                         (long long)n_patch, (long long)s1, (long long)s2, (int)lattice, (long long)plane_k);
        const char* tile_env = std::getenv("FEA_PATCH_TILE");
        if (lattice && (plane_k > (int64_t{64} << 20) || tile_env)) {
            const int T = tile_env ? std::max(1, std::atoi(tile_env)) : 16;
            const std::vector<int32_t> seq = tiled_sequence(n_patch, s1, s2, T);
            std::vector<int32_t> m2(members.size());
            for (int64_t q = 0; q < n_patch; ++q)
                std::copy(members.begin() + static_cast<int64_t>(seq[q]) * P,
                          members.begin() + static_cast<int64_t>(seq[q] + 1) * P, m2.begin() + q * P);
            members.swap(m2);
        }
    }
    mark("lattice + tiles");
    d_mem.alloc(members.size() * 4);
    FEA_CK(cudaMemcpyAsync(d_mem.p, members.data(), members.size() * 4, cudaMemcpyHostToDevice, s));
    FEA_CK(cudaStreamSynchronize(s));
    }
    // per patch: rows, pairs, element pair indices - on the device (k_patch_tables): a count pass,
    // two exclusive scans for the row and pair offsets, a fill pass
    DevBuf d_nr, d_np, d_ro, d_po, d_mx;
    d_nr.alloc((n_patch + 1) * 8);
    d_np.alloc((n_patch + 1) * 8);
    d_ro.alloc((n_patch + 1) * 8);
    d_po.alloc((n_patch + 1) * 8);
    d_mx.alloc(16);
    FEA_CK(cudaMemsetAsync(d_nr.p, 0, d_nr.bytes, s));
    FEA_CK(cudaMemsetAsync(d_np.p, 0, d_np.bytes, s));
    FEA_CK(cudaMemsetAsync(d_mx.p, 0, 16, s));
    const unsigned pt_blocks = grid_for(n_patch * 32, kPtWarps * 32);
    k_patch_tables<false><<<pt_blocks, kPtWarps * 32, 0, s>>>(
        d_mem.as<int32_t>(), n_patch, p->elem_krow.as<int32_t>(), p->conn_k.as<int32_t>(), p->posE.as<uint8_t>(),
        p->nptr.as<int64_t>(), p->node_begin, p->n_own, p->d, d_nr.as<int64_t>(), d_np.as<int64_t>(), nullptr, nullptr,
        0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    FEA_CK(cudaGetLastError());
    k_max2_i64<<<grid_for(n_patch, 256), 256, 0, s>>>(d_nr.as<int64_t>(), d_np.as<int64_t>(), n_patch,
                                                      d_mx.as<unsigned long long>());
    exclusive_sum(d_nr.as<int64_t>(), d_ro.as<int64_t>(), n_patch + 1, s);
    exclusive_sum(d_np.as<int64_t>(), d_po.as<int64_t>(), n_patch + 1, s);
    unsigned long long h_mx[2] = {0, 0};
    int64_t tot_rows = 0, tot_pairs = 0;
    FEA_CK(cudaMemcpyAsync(h_mx, d_mx.p, 16, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(&tot_rows, d_ro.as<int64_t>() + n_patch, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(&tot_pairs, d_po.as<int64_t>() + n_patch, 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    FEA_REQUIRE(tot_pairs < (int64_t{1} << 31) && tot_rows < (int64_t{1} << 31), FEA_ERR_INVALID,
                "internal: patch tables too large");
    const int max_pairs = static_cast<int>(h_mx[1]);
    p->pk_hdr.alloc(std::max<int64_t>(n_patch, 1) * 16);
    p->pk_krow.alloc(static_cast<size_t>(n_patch) * P * 4);
    p->pk_cidx.alloc(static_cast<size_t>(n_patch) * P * NN * 2);
    p->pk_rows.alloc(std::max<int64_t>(tot_rows, 1) * 8);
    p->pk_pairs.alloc(std::max<int64_t>(tot_pairs, 1) * 2);
    p->pk_rowpair.alloc(std::max<int64_t>(tot_rows, 1) * 4);
    FEA_CK(cudaMemsetAsync(p->pk_cidx.p, 0xff, p->pk_cidx.bytes, s));
    k_patch_tables<true><<<pt_blocks, kPtWarps * 32, 0, s>>>(
        d_mem.as<int32_t>(), n_patch, p->elem_krow.as<int32_t>(), p->conn_k.as<int32_t>(), p->posE.as<uint8_t>(),
        p->nptr.as<int64_t>(), p->node_begin, p->n_own, p->d, nullptr, nullptr, d_ro.as<int64_t>(), d_po.as<int64_t>(),
        max_pairs, p->pk_hdr.as<int4>(), p->pk_krow.as<int32_t>(), p->pk_cidx.as<uint16_t>(), p->pk_rows.as<int64_t>(),
        p->pk_rowpair.as<int32_t>(), p->pk_pairs.as<uint16_t>());
    FEA_CK(cudaGetLastError());
    FEA_CK(cudaStreamSynchronize(s));
    mark("patch tables (device)");
    p->pk_max_pairs = max_pairs;
    p->pk_n = n_patch;
}

// Strips of k_atomic_strip (npe = 4, d = 1, byte positions, no repeated nodes): kStripElems
// consecutive elements of the atomic visit order (on a mesh whose consecutive elements share
// nodes — the 6 Kuhn tets of a cube, a row of cubes — 768 element entries fall on ~270 distinct
// slots). A strip's nodes are numbered by first appearance; its distinct (row node, column node)
// pairs are sorted by those local numbers and every pair lists the strip's K entries that feed
// it, ascending (a fixed summation order inside the strip; atomics between strips). That
// structure — list ends, row of each pair, entry offsets: the strip's SHAPE — does not depend on
// the node ids, so strips of a regular mesh share a handful of shapes (de-duplicated by content;
// the kernel reads them from L2), and the per-strip record keeps only what the ids decide: the
// values start of each row node and each pair's position in its row. Host work, once per plan
// (first atomic assembly); both tables have fixed-size records sized by the largest strip.
void build_strips(fea_plan* p, cudaStream_t s) {
    if (p->npe != 4 || p->d != 1 || p->pos_bytes != 1 || p->dup_nodes || p->E == 0 || p->kn.atomic_no_patch ||
        p->kn.atomic_no_strip || p->kn.atomic_legacy || p->sk_n > 0)
        return;
    constexpr int NPE = 4, NN = 16, P = kStripElems;
    const int64_t E = p->E;
    std::vector<int32_t> order(E), krow(E), conn(static_cast<size_t>(p->krows() * NPE));
    std::vector<uint8_t> posE(static_cast<size_t>(E * NN));
    std::vector<int64_t> nptr(static_cast<size_t>(p->n_own + 1));
    FEA_CK(cudaMemcpyAsync(order.data(), p->order.p, E * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(krow.data(), p->elem_krow.p, E * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(conn.data(), p->conn_k.p, conn.size() * 4, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(posE.data(), p->posE.p, posE.size(), cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(nptr.data(), p->nptr.p, nptr.size() * 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    int32_t max_node = 0;
    for (int32_t v : conn) max_node = std::max(max_node, v);
    const int64_t nn = static_cast<int64_t>(max_node) + 1;
    const int64_t n_strip = (E + P - 1) / P;
    struct Strip {
        int64_t rows_off, pairs_off;
        int32_t n_rows, n_pairs, n_ent, n_el, shape;
    };
    struct Shape {
        int64_t pairs_off, ent_off;
        int32_t n_pairs, n_ent;
    };
    std::vector<Strip> st(static_cast<size_t>(n_strip));
    std::vector<int4> hk0(static_cast<size_t>(n_strip));
    std::vector<int32_t> hkrow(static_cast<size_t>(n_strip * P), -1);
    const int long_len = std::getenv("FEA_STRIP_LONG") ? std::atoi(std::getenv("FEA_STRIP_LONG")) : 6;
    // The strips are independent: host threads take contiguous ranges of them, each with its own
    // scratch arrays, outputs and shape table (offsets and shape ids local to the range); the
    // ranges are then concatenated in order and their shapes de-duplicated against each other,
    // so the result does not depend on the number of threads.
    struct Part {
        std::vector<Shape> shapes;
        std::vector<int64_t> rows_all;           // per strip: values start per local node (-1: not owned)
        std::vector<uint8_t> ppos_all;           // per strip: position of each pair in its row
        std::vector<uint16_t> end_all, ent_all;  // per shape: list ends, entry offsets
        std::vector<uint8_t> prow_all;           // per shape: local row node of each pair
        int max_rows = 0, max_pairs = 0, max_ent = 0;
    };
    auto work = [&](int64_t q_begin, int64_t q_end, Part& part) {
        std::vector<Shape>& shapes = part.shapes;
        std::unordered_map<uint64_t, std::vector<int32_t>> by_hash;
        std::vector<int64_t>& rows_all = part.rows_all;
        std::vector<uint8_t>& ppos_all = part.ppos_all;
        std::vector<uint16_t>& end_all = part.end_all;
        std::vector<uint16_t>& ent_all = part.ent_all;
        std::vector<uint8_t>& prow_all = part.prow_all;
        int &max_rows = part.max_rows, &max_pairs = part.max_pairs, &max_ent = part.max_ent;
        std::vector<int32_t> nstamp(nn, -1), nloc(nn, 0);
        std::vector<int32_t> pstamp(static_cast<size_t>(P * NPE) * 256, -1);
        std::vector<uint16_t> pidx(static_cast<size_t>(P * NPE) * 256, 0);
        std::vector<uint8_t> kpos(static_cast<size_t>(P * NPE) * 256, 0);
        std::vector<int32_t> keys, sorted, cnt, cnt2, ord;
        std::vector<uint16_t> epair(P * NN), remap, newidx, t_end, t_ent;
        std::vector<uint8_t> t_prow;
        for (int64_t q = q_begin; q < q_end; ++q) {
            const int n_el = static_cast<int>(std::min<int64_t>(P, E - q * P));
            keys.clear();
            int n_loc = 0;
            bool contig = true;
            const int64_t rows_off = static_cast<int64_t>(rows_all.size());
            for (int k = 0; k < n_el; ++k) {  // local node numbers by first appearance
                const int32_t le = order[q * P + k];
                hkrow[q * P + k] = krow[le];
                contig = contig && krow[le] == krow[order[q * P]] + k;
                for (int a = 0; a < NPE; ++a) {
                    const int32_t v = conn[static_cast<size_t>(krow[le]) * NPE + a];
                    if (nstamp[v] != q) {
                        nstamp[v] = static_cast<int32_t>(q);
                        nloc[v] = n_loc++;
                        const int64_t vo = static_cast<int64_t>(v) - p->node_begin;
                        rows_all.push_back(vo >= 0 && vo < p->n_own ? nptr[vo] : -1);
                    }
                }
            }
            for (int k = 0; k < n_el; ++k) {
                const int32_t le = order[q * P + k];
                const int32_t* cv = conn.data() + static_cast<size_t>(krow[le]) * NPE;
                for (int a = 0; a < NPE; ++a) {
                    const int r = nloc[cv[a]];
                    const bool owned = rows_all[rows_off + r] >= 0;
                    for (int b = 0; b < NPE; ++b) {
                        if (!owned) {  // row not owned: its entries are dropped
                            epair[k * NN + a * NPE + b] = 0xffffu;
                            continue;
                        }
                        const int key = r * 256 + nloc[cv[b]];
                        if (pstamp[key] != q) {
                            pstamp[key] = static_cast<int32_t>(q);
                            pidx[key] = static_cast<uint16_t>(keys.size());
                            kpos[key] = posE[static_cast<size_t>(le) * NN + a * NPE + b];
                            keys.push_back(key);
                        }
                        epair[k * NN + a * NPE + b] = pidx[key];
                    }
                }
            }
            // pairs sorted by (local row, local column); entry lists by counting sort (ascending offset)
            sorted = keys;
            std::sort(sorted.begin(), sorted.end());
            remap.resize(keys.size());
            for (size_t i = 0; i < sorted.size(); ++i) pidx[sorted[i]] = static_cast<uint16_t>(i);
            for (size_t i = 0; i < keys.size(); ++i) remap[i] = pidx[keys[i]];
            const int n_pairs = static_cast<int>(sorted.size());
            cnt.assign(n_pairs + 1, 0);
            int n_ent = 0;
            for (int x = 0; x < n_el * NN; ++x)
                if (epair[x] != 0xffffu) {
                    epair[x] = remap[epair[x]];
                    ++cnt[epair[x] + 1];
                    ++n_ent;
                }
            // thread t of the CTA sums pair t's list, and a warp runs as long as its longest list:
            // the long lists (a node's diagonal collects an entry from each of its elements in the
            // strip, up to 24 on a Kuhn mesh; an edge 1-6) go first, longest first, so they share
            // warps; the short ones keep the (row, column) order, whose neighbours share sectors
            ord.resize(n_pairs);
            for (int i = 0; i < n_pairs; ++i) ord[i] = i;
            std::stable_sort(ord.begin(), ord.end(), [&](int i, int j) {
                const int li = cnt[i + 1], lj = cnt[j + 1];
                if (long_len <= 0) return li > lj;  // FEA_STRIP_LONG=0: all by length
                if ((li > long_len) != (lj > long_len)) return li > long_len;
                return li > long_len ? li > lj : false;
            });
            newidx.resize(n_pairs);
            for (int k = 0; k < n_pairs; ++k) newidx[ord[k]] = static_cast<uint16_t>(k);
            cnt2.assign(n_pairs + 1, 0);
            for (int k = 0; k < n_pairs; ++k) cnt2[k + 1] = cnt2[k] + cnt[ord[k] + 1];
            t_end.resize(n_pairs);
            t_prow.resize(n_pairs);
            t_ent.resize(n_ent);
            const int64_t pairs_off = static_cast<int64_t>(ppos_all.size());
            for (int k = 0; k < n_pairs; ++k) {
                t_end[k] = static_cast<uint16_t>(cnt2[k + 1]);
                t_prow[k] = static_cast<uint8_t>(sorted[ord[k]] >> 8);
                ppos_all.push_back(kpos[sorted[ord[k]]]);
            }
            for (int x = 0; x < n_el * NN; ++x)
                if (epair[x] != 0xffffu) t_ent[cnt2[newidx[epair[x]]]++] = static_cast<uint16_t>(x);
            // shape de-duplication by content
            uint64_t h = 1469598103934665603ull ^ static_cast<uint64_t>(n_pairs) * 1099511628211ull;
            auto mixin = [&](const void* d, size_t n) {
                const unsigned char* c = static_cast<const unsigned char*>(d);
                for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
            };
            mixin(t_end.data(), t_end.size() * 2);
            mixin(t_prow.data(), t_prow.size());
            mixin(t_ent.data(), t_ent.size() * 2);
            int32_t shape = -1;
            for (int32_t c : by_hash[h]) {
                const Shape& sh = shapes[c];
                if (sh.n_pairs == n_pairs && sh.n_ent == n_ent &&
                    std::memcmp(end_all.data() + sh.pairs_off, t_end.data(), n_pairs * 2) == 0 &&
                    std::memcmp(prow_all.data() + sh.pairs_off, t_prow.data(), n_pairs) == 0 &&
                    std::memcmp(ent_all.data() + sh.ent_off, t_ent.data(), n_ent * 2) == 0) {
                    shape = c;
                    break;
                }
            }
            if (shape < 0) {
                shape = static_cast<int32_t>(shapes.size());
                shapes.push_back({static_cast<int64_t>(end_all.size()), static_cast<int64_t>(ent_all.size()), n_pairs, n_ent});
                end_all.insert(end_all.end(), t_end.begin(), t_end.end());
                prow_all.insert(prow_all.end(), t_prow.begin(), t_prow.end());
                ent_all.insert(ent_all.end(), t_ent.begin(), t_ent.end());
                by_hash[h].push_back(shape);
            }
            st[q] = {rows_off, pairs_off, n_loc, n_pairs, n_ent, n_el, shape};
            hk0[q] = make_int4(contig ? krow[order[q * P]] : -1, n_el, shape, 0);
            max_rows = std::max(max_rows, n_loc);
            max_pairs = std::max(max_pairs, n_pairs);
            max_ent = std::max(max_ent, n_ent);
        }
    };
    const int n_thr = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({int64_t{16}, static_cast<int64_t>(std::thread::hardware_concurrency()), n_strip / 1024})));
    std::vector<Part> parts(static_cast<size_t>(n_thr));
    std::vector<int64_t> cut(static_cast<size_t>(n_thr) + 1);
    for (int t = 0; t <= n_thr; ++t) cut[t] = n_strip * t / n_thr;
    {
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(static_cast<size_t>(n_thr));
        auto run = [&](int t) {
            try {
                work(cut[t], cut[t + 1], parts[t]);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        };
        for (int t = 1; t < n_thr; ++t) pool.emplace_back(run, t);
        run(0);
        for (std::thread& th : pool) th.join();
        for (const std::exception_ptr& e : errs)
            if (e) std::rethrow_exception(e);
    }
    // concatenate the ranges; shapes de-duplicated by content across ranges
    std::vector<Shape> shapes;
    std::vector<int64_t> rows_all;
    std::vector<uint8_t> ppos_all, prow_all;
    std::vector<uint16_t> end_all, ent_all;
    int max_rows = 0, max_pairs = 0, max_ent = 0;
    for (int t = 0; t < n_thr; ++t) {
        Part& pt = parts[t];
        std::vector<int32_t> map(pt.shapes.size());
        for (size_t c = 0; c < pt.shapes.size(); ++c) {
            const Shape& sh = pt.shapes[c];
            int32_t g = -1;
            for (size_t k = 0; k < shapes.size() && g < 0; ++k)
                if (shapes[k].n_pairs == sh.n_pairs && shapes[k].n_ent == sh.n_ent &&
                    std::memcmp(end_all.data() + shapes[k].pairs_off, pt.end_all.data() + sh.pairs_off, sh.n_pairs * 2) == 0 &&
                    std::memcmp(prow_all.data() + shapes[k].pairs_off, pt.prow_all.data() + sh.pairs_off, sh.n_pairs) == 0 &&
                    std::memcmp(ent_all.data() + shapes[k].ent_off, pt.ent_all.data() + sh.ent_off, sh.n_ent * 2) == 0)
                    g = static_cast<int32_t>(k);
            if (g < 0) {
                g = static_cast<int32_t>(shapes.size());
                shapes.push_back({static_cast<int64_t>(end_all.size()), static_cast<int64_t>(ent_all.size()), sh.n_pairs, sh.n_ent});
                end_all.insert(end_all.end(), pt.end_all.begin() + sh.pairs_off, pt.end_all.begin() + sh.pairs_off + sh.n_pairs);
                prow_all.insert(prow_all.end(), pt.prow_all.begin() + sh.pairs_off, pt.prow_all.begin() + sh.pairs_off + sh.n_pairs);
                ent_all.insert(ent_all.end(), pt.ent_all.begin() + sh.ent_off, pt.ent_all.begin() + sh.ent_off + sh.n_ent);
            }
            map[c] = g;
        }
        const int64_t rows_base = static_cast<int64_t>(rows_all.size()), pairs_base = static_cast<int64_t>(ppos_all.size());
        for (int64_t q = cut[t]; q < cut[t + 1]; ++q) {
            st[q].rows_off += rows_base;
            st[q].pairs_off += pairs_base;
            st[q].shape = map[st[q].shape];
            hk0[q].z = st[q].shape;
        }
        rows_all.insert(rows_all.end(), pt.rows_all.begin(), pt.rows_all.end());
        ppos_all.insert(ppos_all.end(), pt.ppos_all.begin(), pt.ppos_all.end());
        max_rows = std::max(max_rows, pt.max_rows);
        max_pairs = std::max(max_pairs, pt.max_pairs);
        max_ent = std::max(max_ent, pt.max_ent);
        pt = Part{};
    }
    auto a16 = [](int x) { return (x + 15) & ~15; };
    // strip record: header, row starts, pair positions; shape record: list ends, pair rows, entries
    const int off_pos = 16 + a16(8 * max_rows), stride = off_pos + a16(std::max(max_pairs, 1));
    const int off_prow = a16(2 * std::max(max_pairs, 1)), off_ent = off_prow + a16(std::max(max_pairs, 1)),
              sh_stride = off_ent + a16(2 * std::max(max_ent, 1));
    FEA_REQUIRE(static_cast<size_t>(stride) + sh_stride + P * 128 <= 64 * 1024, FEA_ERR_INVALID,
                "internal: strip record too large");
    std::vector<unsigned char> blob(static_cast<size_t>(n_strip) * stride, 0);
    for (int64_t q = 0; q < n_strip; ++q) {
        unsigned char* b = blob.data() + q * stride;
        const int32_t hdr[4] = {st[q].n_pairs, st[q].n_ent, st[q].n_rows, st[q].n_el};
        std::memcpy(b, hdr, 16);
        std::memcpy(b + 16, rows_all.data() + st[q].rows_off, static_cast<size_t>(st[q].n_rows) * 8);
        std::memcpy(b + off_pos, ppos_all.data() + st[q].pairs_off, static_cast<size_t>(st[q].n_pairs));
    }
    std::vector<unsigned char> sblob(shapes.size() * static_cast<size_t>(sh_stride), 0);
    for (size_t c = 0; c < shapes.size(); ++c) {
        unsigned char* b = sblob.data() + c * sh_stride;
        std::memcpy(b, end_all.data() + shapes[c].pairs_off, static_cast<size_t>(shapes[c].n_pairs) * 2);
        std::memcpy(b + off_prow, prow_all.data() + shapes[c].pairs_off, static_cast<size_t>(shapes[c].n_pairs));
        std::memcpy(b + off_ent, ent_all.data() + shapes[c].ent_off, static_cast<size_t>(shapes[c].n_ent) * 2);
    }
    p->sk_meta.alloc(blob.size());
    p->sk_shape.alloc(std::max<size_t>(sblob.size(), 16));
    p->sk_k0.alloc(hk0.size() * 16);
    p->sk_krow.alloc(hkrow.size() * 4);
    FEA_CK(cudaMemcpyAsync(p->sk_meta.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
    if (!sblob.empty()) FEA_CK(cudaMemcpyAsync(p->sk_shape.p, sblob.data(), sblob.size(), cudaMemcpyHostToDevice, s));
    FEA_CK(cudaMemcpyAsync(p->sk_k0.p, hk0.data(), hk0.size() * 16, cudaMemcpyHostToDevice, s));
    FEA_CK(cudaMemcpyAsync(p->sk_krow.p, hkrow.data(), hkrow.size() * 4, cudaMemcpyHostToDevice, s));
    FEA_CK(cudaStreamSynchronize(s));
    p->sk_stride = stride;
    p->sk_off_pos = off_pos;
    p->sk_sh_stride = sh_stride;
    p->sk_off_prow = off_prow;
    p->sk_off_ent = off_ent;
    p->sk_n = n_strip;
    if (std::getenv("FEA_PATCH_DEBUG"))
        std::fprintf(stderr, "strips: n %lld shapes %zu max nodes %d pairs %d entries %d strides %d %d\n",
                     (long long)n_strip, shapes.size(), max_rows, max_pairs, max_ent, stride, sh_stride);
}

// Visit-order metadata of k_atomic_staged (shapes d <= 3, npe in {4, 8}); other shapes, and
// FEA_ATOMIC_LEGACY=1 (A/B), keep k_scatter<atomic>.
void build_atomic_maps(fea_plan* p, cudaStream_t s) {
    const bool shape = (p->d >= 1 && p->d <= 3 && (p->npe == 4 || p->npe == 8)) ||
                       ((p->d == 1 || p->d == 3) && p->npe == 27);  // k_atomic_staged / k_atomic_cta
    if (!shape || p->E == 0 || p->kn.atomic_legacy ||
        static_cast<int64_t>(p->d) * p->max_cnt >= (1 << 20))
        return;
    const int mm = p->m * p->m;
    const int B = mm >= 128 ? 1 : 128 / mm;  // AtomicShape<>::B (k_atomic_cta: 1)
    p->at_E_pad = (p->E + B - 1) / B * B;
    // position rows padded to 16-byte multiples (whole cp.async pieces)
    const int pstr = ((p->npe * p->npe * p->pos_bytes + 15) & ~15) / p->pos_bytes;
    p->at_krow.alloc(p->at_E_pad * 4);
    p->at_rows.alloc(p->at_E_pad * p->npe * 8);
    p->at_pos.alloc(p->at_E_pad * pstr * p->pos_bytes);
    const unsigned g = grid_for(p->at_E_pad, 256);
    if (p->pos_bytes == 1)
        k_atomic_maps<uint8_t><<<g, 256, 0, s>>>(
            p->order.as<int32_t>(), p->elem_krow.as<int32_t>(), p->conn_k.as<int32_t>(), p->nptr.as<int64_t>(),
            p->posE.as<uint8_t>(), p->E, p->at_E_pad, p->npe, p->d, p->node_begin, p->n_own, pstr,
            p->at_krow.as<int32_t>(), p->at_rows.as<int64_t>(), p->at_pos.as<uint8_t>());
    else
        k_atomic_maps<uint16_t><<<g, 256, 0, s>>>(
            p->order.as<int32_t>(), p->elem_krow.as<int32_t>(), p->conn_k.as<int32_t>(), p->nptr.as<int64_t>(),
            p->posE.as<uint16_t>(), p->E, p->at_E_pad, p->npe, p->d, p->node_begin, p->n_own, pstr,
            p->at_krow.as<int32_t>(), p->at_rows.as<int64_t>(), p->at_pos.as<uint16_t>());
    FEA_CK(cudaGetLastError());
    FEA_CK(cudaStreamSynchronize(s));
}

void assemble(fea_plan* p, const double* K, int strategy, double* values, uint32_t flags,
              cudaStream_t s) {
    FEA_REQUIRE(strategy == FEA_ATOMIC || strategy == FEA_DET_SORTED || strategy == FEA_DET_COLOUR,
                FEA_ERR_INVALID, "unknown strategy");
    if (p->miss_e >= 0) {
        char buf[160];
        std::snprintf(buf, sizeof(buf),
                      "assembly hit a coefficient missing from the pattern: element %lld, (%lld, %lld)",
                      static_cast<long long>(p->miss_e), static_cast<long long>(p->miss_r),
                      static_cast<long long>(p->miss_c));
        throw Error(FEA_ERR_MISSING_ENTRY, buf);
    }
    FEA_REQUIRE(p->nnz == 0 || values, FEA_ERR_INVALID, "values is NULL");
    FEA_REQUIRE(p->E == 0 || K || p->gen_on, FEA_ERR_INVALID, "K is NULL");
    const bool overwrite = (flags & FEA_OVERWRITE) != 0;
    p->last_launches = 0;
    if (strategy == FEA_DET_COLOUR)
        FEA_REQUIRE(p->has_colouring, FEA_ERR_INVALID,
                    "FEA_DET_COLOUR needs a colouring (fea_plan_set_colouring)");
    if (strategy == FEA_DET_SORTED || (strategy == FEA_DET_COLOUR && !(flags & FEA_COLOUR_PASSES))) {
        // DET_COLOUR as a segmented reduction: within each node the incidences are ordered by
        // (colour, element), so every slot folds its contributions in colour order — exactly
        // the summation order of the per-colour passes of assemble_coloured_vectorized.
        Incidences in{p->adj.as<int32_t>(), p->posA.p};
        if (strategy == FEA_DET_COLOUR) in = Incidences{p->adjC.as<int32_t>(), p->posAC.p};
        if (p->pos_bytes == 1) gather_u8(p, in, K, values, !overwrite, s);
        else gather_u16(p, in, K, values, !overwrite, s);
        return;
    }
    ensure_element_maps(p, s);
    if (overwrite && p->nnz > 0) FEA_CK(cudaMemsetAsync(values, 0, p->nnz * 8, s));
    if (strategy == FEA_ATOMIC) {
        if (p->pos_bytes == 1) scatter_u8(p, K, p->order.as<int32_t>(), p->E, values, true, s);
        else scatter_u16(p, K, p->order.as<int32_t>(), p->E, values, true, s);
        return;
    }
    const int nc = static_cast<int>(p->colour_off.size()) - 1;
    for (int c = 0; c < nc; ++c) {
        const int32_t* list = p->colour_elems.as<int32_t>() + p->colour_off[c];
        const int64_t cnt = p->colour_off[c + 1] - p->colour_off[c];
        if (p->pos_bytes == 1) scatter_u8(p, K, list, cnt, values, false, s);
        else scatter_u16(p, K, list, cnt, values, false, s);
    }
}


// --- end-to-end host path (fea_assemble_host) --------------------------------------------
// The whole K must be on the device before the LAST node of the traversal can be assembled,
// but a node needs only the element matrices of its incident elements. For meshes whose
// element order follows the node order (structured meshes, z-slabs: config 5), the K rows
// the first nodes need arrive first. The host path therefore splits the traversal into W
// windows, uploads K in the chunks each window first needs (prefix max of its incidences'
// K rows), launches window j as soon as its chunk has landed, and downloads window j's values
// (a contiguous range when nodes are traversed in id order) while later chunks are still
// coming in: host->device, kernels and device->host overlap, so one call costs about
// max(K upload, values download) instead of their sum. Meshes without that locality (permuted
// element order: window 0 already needs almost all of K) degrade to one upload, then the
// windows, then the download.

__global__ void k_window_tables(const int32_t* __restrict__ order, const int64_t* __restrict__ adj_ptr,
                                const int32_t* __restrict__ adj, const int64_t* __restrict__ nptr,
                                int64_t n_own, int npe, int64_t win, int n_win, int dd,
                                unsigned long long* __restrict__ kmax, int64_t* __restrict__ voff) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i <= n_win) voff[i] = dd * nptr[i * win < n_own ? i * win : n_own];
    for (int64_t t = i; t < n_own; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = order != nullptr ? order[t] : t;
        int64_t mx = -1;
        for (int64_t a = adj_ptr[v]; a < adj_ptr[v + 1]; ++a) mx = max(mx, static_cast<int64_t>(adj[a] / npe));
        if (mx >= 0) atomicMax(kmax + t / win, static_cast<unsigned long long>(mx + 1));
    }
}

void ensure_windows(fea_plan* p, cudaStream_t s) {
    HostPipe& q = p->pipe;
    if (q.n_win > 0) return;
    const int64_t kb = p->kbytes_required();
    // K chunks of >= 256 MB, at most 32 windows (or the caller's count), windows a multiple of
    // 64 traversal positions
    int64_t n_win = q.want_win > 0 ? q.want_win
                                   : std::min<int64_t>(32, std::max<int64_t>(1, kb / (int64_t{256} << 20)));
    int64_t win = (p->n_own + n_win - 1) / std::max<int64_t>(n_win, 1);
    win = std::max<int64_t>(64, (win + 63) / 64 * 64);
    n_win = std::max<int64_t>(1, (p->n_own + win - 1) / win);
    q.n_win = static_cast<int>(n_win);
    q.t_win.resize(n_win + 1);
    for (int64_t j = 0; j <= n_win; ++j) q.t_win[j] = std::min<int64_t>(j * win, p->n_own);
    q.k_end.assign(n_win, 0);
    q.v_off.assign(n_win + 1, 0);
    q.v_contiguous = p->node_order.p == nullptr;
    if (p->n_own == 0) return;
    DevBuf kmax, voff;
    kmax.alloc(n_win * 8);
    voff.alloc((n_win + 1) * 8);
    FEA_CK(cudaMemsetAsync(kmax.p, 0, n_win * 8, s));
    k_window_tables<<<grid_for(std::max<int64_t>(p->n_own, n_win + 1), 256), 256, 0, s>>>(
        p->node_order.p ? p->node_order.as<int32_t>() : nullptr, p->adj_ptr.as<int64_t>(), p->adj.as<int32_t>(),
        p->nptr.as<int64_t>(), p->n_own, p->npe, win, static_cast<int>(n_win), p->d * p->d,
        kmax.as<unsigned long long>(), voff.as<int64_t>());
    FEA_CK(cudaGetLastError());
    std::vector<unsigned long long> hk(n_win);
    FEA_CK(cudaMemcpyAsync(hk.data(), kmax.p, n_win * 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaMemcpyAsync(q.v_off.data(), voff.p, (n_win + 1) * 8, cudaMemcpyDeviceToHost, s));
    FEA_CK(cudaStreamSynchronize(s));
    int64_t run = 0;
    for (int64_t j = 0; j < n_win; ++j) {
        run = std::max<int64_t>(run, static_cast<int64_t>(hk[j]));
        q.k_end[j] = run;
    }
}

void assemble_host_pipelined(fea_plan* p, const double* K_host, int32_t strategy, double* values_host,
                             uint32_t flags, cudaStream_t sc) {
    const size_t kb = static_cast<size_t>(p->kbytes_required());
    const size_t vb = static_cast<size_t>(p->nnz) * 8;
    FEA_REQUIRE(kb == 0 || K_host, FEA_ERR_INVALID, "K is NULL");
    FEA_REQUIRE(vb == 0 || values_host, FEA_ERR_INVALID, "values is NULL");
    if (p->stage_K.bytes < kb) p->stage_K.alloc(kb);
    if (p->stage_V.bytes < vb) p->stage_V.alloc(vb);
    double* dK = p->stage_K.as<double>();
    double* dV = p->stage_V.as<double>();
    const bool acc = !(flags & FEA_OVERWRITE);
    HostPipe& q = p->pipe;
    // windows only for the segmented-reduction routes whose kernel takes them (asked after the
    // kernel's lazy tables are built: the query call launches nothing)
    bool windows = false;
    if (strategy == FEA_DET_SORTED || (strategy == FEA_DET_COLOUR && !(flags & FEA_COLOUR_PASSES))) {
        ensure_windows(p, sc);
        if (q.n_win > 1) {
            p->win_query = true;
            p->win_ok = false;
            try {
                assemble(p, dK, strategy, dV, flags, sc);
            } catch (...) {
                p->win_query = false;
                throw;
            }
            p->win_query = false;
            windows = p->win_ok;
        }
    }
    const int nw = windows ? q.n_win : 1;
    q.ensure_events(2 * nw + 1);
    cudaEvent_t* ev_in = q.ev.data();
    cudaEvent_t* ev_done = q.ev.data() + nw;
    cudaEvent_t ev_start = q.ev[2 * nw];
    FEA_CK(cudaEventRecord(ev_start, sc));  // copies start behind the caller's queued work
    FEA_CK(cudaStreamWaitEvent(q.sin, ev_start, 0));
    FEA_CK(cudaStreamWaitEvent(q.sout, ev_start, 0));
    const int64_t mm = static_cast<int64_t>(p->m) * p->m;
    int32_t launches = 0;
    struct WinReset {
        fea_plan* p;
        ~WinReset() { p->win_n = -1; p->win_t0 = 0; }
    } wr{p};
    try {
        if (!windows) {
            if (kb) FEA_CK(cudaMemcpyAsync(dK, K_host, kb, cudaMemcpyHostToDevice, q.sin));
            if (acc && vb) FEA_CK(cudaMemcpyAsync(dV, values_host, vb, cudaMemcpyHostToDevice, q.sin));
            FEA_CK(cudaEventRecord(ev_in[0], q.sin));
            FEA_CK(cudaStreamWaitEvent(sc, ev_in[0], 0));
            assemble(p, dK, strategy, dV, flags, sc);
            launches = p->last_launches;
            FEA_CK(cudaEventRecord(ev_done[0], sc));
            FEA_CK(cudaStreamWaitEvent(q.sout, ev_done[0], 0));
            if (vb) FEA_CK(cudaMemcpyAsync(values_host, dV, vb, cudaMemcpyDeviceToHost, q.sout));
        } else {
            const bool vc = q.v_contiguous;
            if (acc && !vc && vb) FEA_CK(cudaMemcpyAsync(dV, values_host, vb, cudaMemcpyHostToDevice, q.sin));
            int64_t k_done = 0;
            for (int j = 0; j < nw; ++j) {
                const int64_t k_hi = q.k_end[j];
                if (k_hi > k_done) {
                    FEA_CK(cudaMemcpyAsync(dK + k_done * mm, K_host + k_done * mm,
                                           static_cast<size_t>(k_hi - k_done) * mm * 8, cudaMemcpyHostToDevice,
                                           q.sin));
                    k_done = k_hi;
                }
                const int64_t v0 = q.v_off[j], v1 = q.v_off[j + 1];
                if (acc && vc && v1 > v0)
                    FEA_CK(cudaMemcpyAsync(dV + v0, values_host + v0, (v1 - v0) * 8, cudaMemcpyHostToDevice, q.sin));
                FEA_CK(cudaEventRecord(ev_in[j], q.sin));
                FEA_CK(cudaStreamWaitEvent(sc, ev_in[j], 0));
                p->win_t0 = q.t_win[j];
                p->win_n = q.t_win[j + 1] - q.t_win[j];
                assemble(p, dK, strategy, dV, flags, sc);
                launches += p->last_launches;
                FEA_CK(cudaEventRecord(ev_done[j], sc));
                if (vc && v1 > v0) {
                    FEA_CK(cudaStreamWaitEvent(q.sout, ev_done[j], 0));
                    FEA_CK(cudaMemcpyAsync(values_host + v0, dV + v0, (v1 - v0) * 8, cudaMemcpyDeviceToHost, q.sout));
                }
            }
            p->win_n = -1;
            p->win_t0 = 0;
            if (!vc && vb) {
                FEA_CK(cudaStreamWaitEvent(q.sout, ev_done[nw - 1], 0));
                FEA_CK(cudaMemcpyAsync(values_host, dV, vb, cudaMemcpyDeviceToHost, q.sout));
            }
        }
        FEA_CK(cudaStreamSynchronize(q.sin));
        FEA_CK(cudaStreamSynchronize(sc));
        FEA_CK(cudaStreamSynchronize(q.sout));
    } catch (...) {
        cudaStreamSynchronize(q.sin);
        cudaStreamSynchronize(sc);
        cudaStreamSynchronize(q.sout);
        throw;
    }
    p->last_launches = launches;
}

}  // namespace feagpu

using namespace feagpu;

namespace {
template <class F>
fea_status guarded_n(F&& f) {
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

fea_status fea_assemble(fea_plan* plan, const double* K, int32_t strategy, double* values,
                        uint32_t flags, void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(plan, FEA_ERR_INVALID, "plan is NULL");
        DeviceScope ds(plan->device);
        assemble(plan, K, strategy, values, flags, static_cast<cudaStream_t>(stream));
    });
}

fea_status fea_assemble_host(fea_plan* plan, const double* K_host, int32_t strategy,
                             double* values_host, uint32_t flags, void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(plan, FEA_ERR_INVALID, "plan is NULL");
        DeviceScope ds(plan->device);
        assemble_host_pipelined(plan, K_host, strategy, values_host, flags, static_cast<cudaStream_t>(stream));
    });
}

// Repeated end-to-end assemblies (new element matrices each step, e.g. Newton or time
// steps): step i's K host->device copy overlaps step i-1's values device->host copy and
// kernel (full-duplex PCIe, separate copy streams), with two device staging slots.
// Every step still moves its whole K in and its whole values array out. Synchronous.
fea_status fea_assemble_host_batch(fea_plan* plan, const double* const* K_hosts, int32_t strategy,
                                   double* const* values_hosts, int32_t n_steps, uint32_t flags,
                                   void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(plan && n_steps >= 0 && (n_steps == 0 || (K_hosts && values_hosts)),
                    FEA_ERR_INVALID, "bad arguments");
        DeviceScope ds(plan->device);
        cudaStream_t sc = static_cast<cudaStream_t>(stream);
        const size_t kb = static_cast<size_t>(plan->kbytes_required());
        const size_t vb = static_cast<size_t>(plan->nnz) * 8;
        for (int s2 = 0; s2 < 2; ++s2) {
            if (plan->bstage_K[s2].bytes < kb) plan->bstage_K[s2].alloc(kb);
            if (plan->bstage_V[s2].bytes < vb) plan->bstage_V[s2].alloc(vb);
        }
        HostPipe& q = plan->pipe;
        q.ensure_events(6);
        cudaStream_t sin = q.sin, sout = q.sout;
        cudaEvent_t* ev_in = q.ev.data();
        cudaEvent_t* ev_done = q.ev.data() + 2;
        cudaEvent_t* ev_out = q.ev.data() + 4;
        // the copy streams start behind whatever the caller queued on its stream
        FEA_CK(cudaEventRecord(ev_done[0], sc));
        FEA_CK(cudaStreamWaitEvent(sin, ev_done[0], 0));
        FEA_CK(cudaStreamWaitEvent(sout, ev_done[0], 0));
        int32_t launches = 0;
        try {
            for (int32_t i = 0; i < n_steps; ++i) {
                const int sl = i & 1;
                double* dK = plan->bstage_K[sl].as<double>();
                double* dV = plan->bstage_V[sl].as<double>();
                if (i >= 2) {  // slot reuse: kernel i-2 done with K, copy-out i-2 done with values
                    FEA_CK(cudaStreamWaitEvent(sin, ev_done[sl], 0));
                    FEA_CK(cudaStreamWaitEvent(sin, ev_out[sl], 0));
                }
                if (kb) FEA_CK(cudaMemcpyAsync(dK, K_hosts[i], kb, cudaMemcpyHostToDevice, sin));
                if (!(flags & FEA_OVERWRITE) && vb)
                    FEA_CK(cudaMemcpyAsync(dV, values_hosts[i], vb, cudaMemcpyHostToDevice, sin));
                FEA_CK(cudaEventRecord(ev_in[sl], sin));
                FEA_CK(cudaStreamWaitEvent(sc, ev_in[sl], 0));
                assemble(plan, dK, strategy, dV, flags, sc);
                launches += plan->last_launches;
                FEA_CK(cudaEventRecord(ev_done[sl], sc));
                FEA_CK(cudaStreamWaitEvent(sout, ev_done[sl], 0));
                if (vb) FEA_CK(cudaMemcpyAsync(values_hosts[i], dV, vb, cudaMemcpyDeviceToHost, sout));
                FEA_CK(cudaEventRecord(ev_out[sl], sout));
            }
            FEA_CK(cudaStreamSynchronize(sin));
            FEA_CK(cudaStreamSynchronize(sc));
            FEA_CK(cudaStreamSynchronize(sout));
        } catch (...) {
            cudaStreamSynchronize(sin);
            cudaStreamSynchronize(sc);
            cudaStreamSynchronize(sout);
            throw;
        }
        plan->last_launches = launches;
    });
}

fea_status fea_plan_set_host_windows(fea_plan* plan, int32_t n_windows) {
    return guarded_n([&] {
        FEA_REQUIRE(plan && n_windows >= 0, FEA_ERR_INVALID, "bad arguments");
        plan->pipe.want_win = n_windows;
        plan->pipe.n_win = 0;  // rebuilt on the next fea_assemble_host
    });
}

fea_status fea_assemble_seeded(fea_plan* plan, uint64_t seed, int32_t strategy, double* values,
                               uint32_t flags, void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(plan, FEA_ERR_INVALID, "plan is NULL");
        FEA_REQUIRE(strategy == FEA_DET_SORTED || (strategy == FEA_DET_COLOUR && !(flags & FEA_COLOUR_PASSES)),
                    FEA_ERR_INVALID, "the fused supplier runs in the segmented-reduction routes "
                                     "(FEA_DET_SORTED, FEA_DET_COLOUR)");
        DeviceScope ds(plan->device);
        plan->gen_on = true;
        plan->gen_seed = seed;
        try {
            assemble(plan, nullptr, strategy, values, flags, static_cast<cudaStream_t>(stream));
        } catch (...) {
            plan->gen_on = false;
            throw;
        }
        plan->gen_on = false;
    });
}

fea_status fea_fill_seeded_k(double* K, int64_t n, int32_t m, uint64_t seed,
                             const int64_t* elem_ids, void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(n >= 0 && m >= 1 && (n == 0 || K), FEA_ERR_INVALID, "bad arguments");
        if (n == 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        k_fill_k<<<grid_for(n * m * m, 256), 256, 0, s>>>(K, n, m, seed, elem_ids);
        FEA_CK(cudaGetLastError());
    });
}

fea_status fea_exclusive_sum_i64(const int64_t* in, int64_t* out, int64_t n, void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(n >= 0 && (n == 0 || (in && out)), FEA_ERR_INVALID, "bad arguments");
        exclusive_sum(in, out, n, static_cast<cudaStream_t>(stream));
        FEA_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    });
}

fea_status fea_sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
                              int32_t* vals_out, int64_t n, int32_t begin_bit, int32_t end_bit, void* stream) {
    return guarded_n([&] {
        FEA_REQUIRE(n >= 0 && (n == 0 || (keys_in && keys_out && vals_in && vals_out)) && begin_bit >= 0 &&
                        end_bit <= 32 && begin_bit <= end_bit,
                    FEA_ERR_INVALID, "bad arguments");
        radix_sort_pairs(keys_in, keys_out, vals_in, vals_out, n, begin_bit, end_bit,
                         static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
