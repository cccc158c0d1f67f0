// Microbenchmark: the DET_SORTED memory pattern without any arithmetic — per "node",
// read 8 random 576 B chunks of K and write one 1944 B block of values (cfg2 sizes).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
__global__ void pattern(const double* __restrict__ K, const int32_t* __restrict__ chunk_ids,
                        int64_t n_nodes, double* __restrict__ out, int write) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = warp; v < n_nodes; v += nw) {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double2* src = reinterpret_cast<const double2*>(K + (int64_t)chunk_ids[v * 8 + c] * 72);
            double2 a = __ldcs(src + lane);
            acc[c] = a.x + a.y;
            if (lane < 4) { double2 b = __ldcs(src + 32 + lane); acc[c] += b.x + b.y; }
        }
        double s = 0; for (int c = 0; c < 8; ++c) s += acc[c];
        if (write) for (int i = lane; i < 243; i += 32) __stcs(out + v * 243 + i, s + i);
        else if (s == 1.2345) out[0] = s;
    }
}
int main() {
    const int64_t E = 262144, n_nodes = 274625, chunks = E * 8;
    double* K; cudaMalloc(&K, E * 576 * 8); cudaMemset(K, 0, E * 576 * 8);
    double* out; cudaMalloc(&out, n_nodes * 243 * 8);
    std::vector<int32_t> ids(n_nodes * 8);
    std::mt19937_64 rng(1);
    for (auto& x : ids) x = (int32_t)(rng() % chunks);
    int32_t* d_ids; cudaMalloc(&d_ids, ids.size() * 4);
    cudaMemcpy(d_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int write : {0, 1}) for (int bs : {128, 256}) for (int grid : {148 * 8, 148 * 16, 148 * 32}) {
        pattern<<<grid, bs>>>(K, d_ids, n_nodes, out, write);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) pattern<<<grid, bs>>>(K, d_ids, n_nodes, out, write);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        double bytes = n_nodes * 8.0 * 576 + (write ? n_nodes * 243.0 * 8 : 0);
        printf("write=%d bs=%d grid=%d: %.3f ms  %.0f GB/s\n", write, bs, grid, ms, bytes / ms / 1e6);
    }
    return 0;
}
