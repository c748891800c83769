// ex2_probe.cu -- measured accuracy of the MUFU exponential on this GPU (a development
// probe, not product code): ex2.approx.ftz.f32 and ex2.approx.ftz.bf16x2 against the
// fp64 exp2 over a dense grid of arguments in [-32, 0] (every fp32 value in sub-ranges),
// reporting the max and mean relative error (the mean says whether the unit is biased).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ex2_probe ex2_probe.cu && ./ex2_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b(uint32_t x) { uint32_t y; asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

struct Acc { double sum, sabs, mx; unsigned long long n; };

__global__ void probe(float lo, float hi, uint64_t n, Acc *out, int bf) {
    double s = 0, sa = 0, mx = 0; unsigned long long cnt = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float x = lo + (hi - lo) * (float)((double)i / (double)n);
        double ex, got;
        if (bf) {
            __nv_bfloat16 xb = __float2bfloat16_rn(x);
            float xr = __bfloat162float(xb);
            uint32_t w = (uint32_t)__bfloat16_as_ushort(xb) | ((uint32_t)__bfloat16_as_ushort(xb) << 16);
            uint32_t y = ex2b(w);
            got = (double)__uint_as_float(y << 16);
            ex = exp2((double)xr);
        } else {
            got = (double)ex2f(x);
            ex = exp2((double)x);
        }
        if (ex < 1e-37) continue;
        double r = (got - ex) / ex;
        s += r; sa += fabs(r); mx = fmax(mx, fabs(r)); cnt++;
    }
    atomicAdd(&out->sum, s); atomicAdd(&out->sabs, sa); atomicAdd(&out->n, cnt);
    unsigned long long* m = (unsigned long long*)&out->mx;
    unsigned long long old = *m, assumed;
    do { assumed = old; if (__longlong_as_double(assumed) >= mx) break;
         old = atomicCAS(m, assumed, __double_as_longlong(mx)); } while (assumed != old);
}

int main() {
    Acc *d; cudaMalloc(&d, sizeof(Acc));
    const float ranges[][2] = {{-32.f, 0.f}, {-1.f, 0.f}, {-0.01f, 0.f}, {0.f, 1.f}, {-126.f, -100.f}};
    for (int bf = 0; bf < 2; ++bf)
        for (auto &r : ranges) {
            cudaMemset(d, 0, sizeof(Acc));
            probe<<<148 * 8, 256>>>(r[0], r[1], 1ull << 28, d, bf);
            Acc h; cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
            printf("{\"op\": \"%s\", \"lo\": %g, \"hi\": %g, \"n\": %llu, \"mean_rel\": %.3e, \"mean_abs_rel\": %.3e, \"max_rel\": %.3e}\n",
                   bf ? "ex2.approx.ftz.bf16x2" : "ex2.approx.ftz.f32", r[0], r[1], h.n, h.sum / h.n, h.sabs / h.n, h.mx);
        }
    return 0;
}
