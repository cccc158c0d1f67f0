// DRAM fetch granularity probe: read one 32 B sector (sector s) of every 128 B line of a
// buffer far larger than L2, then the other sectors in a second pass. ncu's dram__bytes_read
// per pass shows whether an L2 miss fetches 32 B, 64 B or the whole line.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_sector(const double* __restrict__ p, long n_lines, int sector, double* out) {
    double s = 0;
    for (long l = blockIdx.x * (long)blockDim.x + threadIdx.x; l < n_lines; l += (long)gridDim.x * blockDim.x)
        s += __ldcg(p + l * 16 + sector * 4);
    if (s == 12345.0) out[0] = s;
}
int main() {
    const long bytes = 2L << 30, n_lines = bytes / 128;
    double *p, *out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(p, 0, bytes);
    for (int sec = 0; sec < 4; ++sec) k_sector<<<148 * 16, 256>>>(p, n_lines, sec, out);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
}
