// L2 capacity probe: `passes` sweeps over a buffer of `mb` MB by every SM, the CTA -> chunk
// assignment rotated by a prime stride each pass (so a chunk is re-read from the other die's
// SMs too); ncu's dram__bytes_read.sum / (passes x size) says how much of the re-reads L2
// absorbed.  nvcc -gencode arch=compute_100a,code=sm_100a -o l2_probe l2_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void sweep(const uint4 *buf, size_t n_vec, int passes, int rotate, unsigned long long *sink) {
    const size_t chunk = (n_vec + gridDim.x - 1) / gridDim.x;
    uint32_t acc = 0;
    for (int p = 0; p < passes; ++p) {
        const size_t b = rotate ? (blockIdx.x + (size_t)p * 37) % gridDim.x : blockIdx.x;
        const size_t lo = b * chunk, hi = min(n_vec, lo + chunk);
        for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            uint4 v;
            asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncthreads();
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char **argv) {
    const int rotate = argc > 1 ? atoi(argv[1]) : 1;
    const int sizes[] = {24, 40, 56, 64, 72, 88, 104, 120};
    uint4 *buf;
    unsigned long long *sink;
    cudaMalloc(&buf, 128ull << 20);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, 128ull << 20);
    for (int s : sizes) {
        const size_t n_vec = ((size_t)s << 20) / 16;
        sweep<<<148 * 2, 512>>>(buf, n_vec, 8, rotate, sink);
        cudaDeviceSynchronize();
        printf("size_mb %d passes 8 rotate %d\n", s, rotate);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
