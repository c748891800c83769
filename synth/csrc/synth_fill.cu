// synth_fill.cu -- TEST/BENCH INPUT GENERATOR (device twin of synth/gen.py's
// LogitsSpec).  Holds none of the method's arithmetic: it only fills
//   z[k, v] = bf16_rn(base[v] + scale * c((row_begin + k) mod period, v)),
//   c = (sum of the four 16-bit lanes of SplitMix64 draw #(row*V + v)) - 131070,
// with single-rounding float32 ops (__fmul_rn / __fadd_rn, no FMA), so it is
// bit-identical to the numpy generator.  Padding columns [V, ld) get a NaN
// pattern so any read of them by a consumer shows up in its results.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t bf16_rn(float x) {
    const uint32_t b = __float_as_uint(x);
    return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

__global__ void fill_kernel(uint16_t *out, int64_t n_rows, int64_t row_begin, int64_t period,
                            int32_t V, int64_t ld, uint64_t key, const float *base, float scale) {
    const int64_t total = n_rows * ld;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx / ld;
        const int64_t v = idx - k * ld;
        if (v >= V) {
            out[idx] = 0x7FC1;  // NaN in padding
            continue;
        }
        const uint64_t row = (uint64_t)((row_begin + k) % period);
        const uint64_t h = mix64(key + ((row * (uint64_t)V + (uint64_t)v) + 1ull) * 0x9E3779B97F4A7C15ull);
        const int64_t c = (int64_t)((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) +
                                    (h >> 48)) - 131070;
        const float a = __fmul_rn((float)c, scale);
        out[idx] = bf16_rn(__fadd_rn(base[v], a));
    }
}

}  // namespace

extern "C" int synth_fill_logits(uint16_t *out, int64_t n_rows, int64_t row_begin, int64_t period,
                                 int32_t V, int64_t ld, uint64_t key, const float *base,
                                 float scale, void *stream) {
    if (n_rows <= 0) return 0;
    const int64_t total = n_rows * ld;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, n_rows, row_begin, period,
                                                                    V, ld, key, base, scale);
    return (int)cudaGetLastError();
}
