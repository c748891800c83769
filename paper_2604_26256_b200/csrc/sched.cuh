// sched.cuh -- dynamic work-unit scheduling for the persistent tcgen05 GEMM kernels
// (lmhead.cu, lmhead_dx.cu).
//
// With a static round-robin (CTA pair g takes units g, g + grid, ...), the pairs drift apart
// over a long launch. The units running at one time then span several raster waves, and
// the operand tiles they share leave L2 between their users. That costs DRAM traffic, and
// under the 1 kW cap it costs clock. Here the pair leader's TMA producer
// thread takes the next unit from a global atomic counter when it is ready to load it, so
// the running units always form one contiguous window of the raster order.
//
// The unit id goes to the pair's other roles through a DEPTH-deep queue in shared memory:
//   fetch (leader's producer):  wait empty[s]; u = atomicAdd(counter, 1) (-1 past the end);
//                               ids[s] = u here and in the peer CTA (st.shared::cluster);
//                               arrive on full[s] here and, release.cluster, in the peer
//   next (every other role):    wait full[s] (acquire.cluster in the peer); u = ids[s];
//                               arrive on the leader's empty[s]
// The consumers are the leader's MMA thread and 4 epilogue warps, plus the peer's producer
// thread and 4 epilogue warps for CTA pairs: empty[s] counts 5 (CG = 1) or 10 (CG = 2)
// arrivals. A role stops after it has read -1.
//
// (With counter == nullptr the same queue carries the static round robin.)
// The counter must be 0 at launch: each launcher zeroes a slot of a small per-file array
// (cudaMemsetAsync on the launch stream), rotating through the slots so that launches that
// overlap on other streams get their own counter.
#pragma once
#include <stdint.h>

#include <atomic>

#include "common.cuh"
#include "tc.cuh"

namespace grpo {
namespace sched {

constexpr int DEPTH = 4;
constexpr int N_COUNTERS = 64;

struct __align__(8) Queue {
    uint64_t full[DEPTH];
    uint64_t empty[DEPTH];
    int32_t ids[DEPTH];
};

template <int CG>
__device__ __forceinline__ void init(Queue *q) {
    for (int s = 0; s < DEPTH; ++s) {
        mbar_init(q->full + s, 1);
        mbar_init(q->empty + s, CG == 2 ? 10 : 5);
    }
}

// the pair leader's TMA producer thread, use i of the queue; counter == nullptr: the static
// round robin instead (unit = pair + i * pairs), for units so long that the pairs' phases
// matter more than their order (dX: K = the vocabulary; once the dynamic order has spread
// the pairs' start times, the pairs that share a k-slice of A or B are at different k)
template <int CG>
__device__ __forceinline__ int fetch(Queue *q, int i, int32_t *counter, int n_units) {
    const int s = i % DEPTH;
    const uint32_t ph = (uint32_t)(i / DEPTH) & 1u;
    mbar_wait(q->empty + s, ph ^ 1u);
    int u;
    if (counter) {
        u = atomicAdd(counter, 1);
    } else {
        const int pair = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
        const int pairs = CG == 2 ? (int)ncluster_x() : (int)gridDim.x;
        u = pair + i * pairs;
    }
    if (u >= n_units) u = -1;
    *reinterpret_cast<volatile int32_t *>(q->ids + s) = u;
    if (CG == 2) {
        const uint32_t r = mapa_shared(smem_u32(q->ids + s), 1u);
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(r), "r"(u) : "memory");
        tc::mbar_arrive_remote(q->full + s, 1u);  // release.cluster: the store above first
    }
    mbar_arrive(q->full + s);
    return u;
}

// every other role, use i of the queue (crank = this CTA's rank in the pair)
template <int CG>
__device__ __forceinline__ int next(Queue *q, int i, uint32_t crank) {
    const int s = i % DEPTH;
    const uint32_t ph = (uint32_t)(i / DEPTH) & 1u;
    if (CG == 2 && crank != 0) mbar_wait_cluster(q->full + s, ph);
    else mbar_wait(q->full + s, ph);
    const int u = *reinterpret_cast<volatile int32_t *>(q->ids + s);
    if (CG == 2 && crank != 0) tc::mbar_arrive_remote(q->empty + s, 0u);
    else mbar_arrive(q->empty + s);
    return u;
}

// host: the next counter slot of a file's array (`base` = cudaGetSymbolAddress of its
// __device__ int32_t[N_COUNTERS]), zeroed on the launch stream
inline cudaError_t take_counter(int32_t *base, cudaStream_t s, int32_t **out) {
    static std::atomic<unsigned> rot{0};
    int32_t *c = base + (rot.fetch_add(1u) % N_COUNTERS);
    *out = c;
    return cudaMemsetAsync(c, 0, sizeof(int32_t), s);
}

}  // namespace sched
}  // namespace grpo
