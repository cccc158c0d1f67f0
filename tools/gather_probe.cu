// Microbenchmark: how fast can B200 gather the cfg2 K chunks (576 B, random order)?
// Reads K in node-adjacency order (the DET_SORTED access pattern) and in element order.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
__global__ void gather_chunks(const double* __restrict__ K, const int32_t* __restrict__ chunk_ids,
                              int64_t n_chunks, int words16, double* out) {
    // one warp per chunk-group of 1; lanes read 16B words
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    double acc = 0;
    for (int64_t c = warp; c < n_chunks; c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double2* src = reinterpret_cast<const double2*>(K + (int64_t)chunk_ids[c] * words16 * 2);
        for (int w = lane; w < words16; w += 32) { double2 v = __ldcs(src + w); acc += v.x + v.y; }
    }
    if (acc == 12345.678) out[0] = acc;
}
int main() {
    const int64_t E = 262144; const int npe = 8; const int dm = 72; const int words16 = dm * 8 / 16;
    const int64_t n_chunks = E * npe;
    double* K; cudaMalloc(&K, E * 576 * 8); cudaMemset(K, 0, E * 576 * 8);
    double* out; cudaMalloc(&out, 8);
    std::vector<int32_t> ids(n_chunks);
    for (int64_t i = 0; i < n_chunks; ++i) ids[i] = (int32_t)i;
    int32_t* d_ids; cudaMalloc(&d_ids, n_chunks * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name) {
        cudaMemcpy(d_ids, ids.data(), n_chunks * 4, cudaMemcpyHostToDevice);
        for (int bs : {128, 256}) for (int grid : {148 * 8, 148 * 16, 148 * 32}) {
            gather_chunks<<<grid, bs>>>(K, d_ids, n_chunks, words16, out);
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) gather_chunks<<<grid, bs>>>(K, d_ids, n_chunks, words16, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
            printf("%-28s bs=%d grid=%d: %.3f ms  %.0f GB/s\n", name, bs, grid, ms, E * 576 * 8 / ms / 1e6);
        }
    };
    run("sequential chunks");
    std::mt19937_64 rng(1); std::shuffle(ids.begin(), ids.end(), rng);
    run("random chunks");
    // random elements, chunks of an element consecutive
    std::vector<int32_t> perm(E); for (int64_t i = 0; i < E; ++i) perm[i] = (int32_t)i;
    std::shuffle(perm.begin(), perm.end(), rng);
    for (int64_t e = 0; e < E; ++e) for (int a2 = 0; a2 < npe; ++a2) ids[e * npe + a2] = perm[e] * npe + a2;
    run("random elements, 8 chunks");
    return 0;
}
