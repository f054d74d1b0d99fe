// handoff.cu -- microbenchmark: round-trip latency of an mbarrier hand-off between the two CTAs
// of a cluster (remote mbarrier.arrive.shared::cluster + local wait), and of a tcgen05.commit
// multicast with no MMA outstanding, with the wait primitives the kernels use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2106_12169_b200/csrc handoff.cu -o handoff
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"

using namespace apnn::sm100;

__device__ __forceinline__ bool test_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool try_wait_hint(uint32_t addr, uint32_t parity, uint32_t ns) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(addr), "r"(parity), "r"(ns) : "memory");
    return ok != 0;
}

template <int MODE>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
    const uint32_t a = smem_u32(bar);
    if (MODE == 0) { while (!mbar_try_wait(a, ph)) {} }
    else if (MODE == 1) { while (!test_wait(a, ph)) {} }
    else { while (!try_wait_hint(a, ph, 20)) {} }
}

// ping-pong: CTA 0 thread arrives on CTA 1's barrier, CTA 1 waits then arrives on CTA 0's barrier
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, unsigned long long* out) {
    __shared__ uint64_t bar;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    cluster_sync();
    const uint32_t peer = mapa(smem_u32(&bar), rank ^ 1);
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; i++) {
            if (rank == 0) {
                mbar_arrive_cluster(peer);
                wait<MODE>(&bar, i & 1);
            } else {
                wait<MODE>(&bar, i & 1);
                mbar_arrive_cluster(peer);
            }
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[MODE] = (t1 - t0) / iters;
    __syncthreads();
    cluster_sync();
}

// local ping-pong inside one CTA between warp 0 and warp 1 (reference)
template <int MODE>
__global__ void local_pingpong(int iters, unsigned long long* out) {
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
    __syncthreads();
    unsigned long long t0 = clock64();
    const int w = threadIdx.x / 32;
    if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < iters; i++) {
            if (w == 0) { mbar_arrive(&bar[1]); wait<MODE>(&bar[0], i & 1); }
            else { wait<MODE>(&bar[1], i & 1); mbar_arrive(&bar[0]); }
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[4 + MODE] = (t1 - t0) / iters;
}

// tcgen05.commit (no MMA outstanding) -> mbarrier -> wait, single CTA
__global__ void commit_lat(int iters, unsigned long long* out) {
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc<32>(&holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; i++) {
            mma_commit(&bar);
            wait<0>(&bar, i & 1);
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[8] = (t1 - t0) / iters;
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(holder, 32);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16 * sizeof(unsigned long long));
    cudaMemset(d, 0, 16 * sizeof(unsigned long long));
    const int it = 10000;
    pingpong<0><<<2, 64>>>(it, d);
    pingpong<1><<<2, 64>>>(it, d);
    pingpong<2><<<2, 64>>>(it, d);
    local_pingpong<0><<<1, 64>>>(it, d);
    local_pingpong<1><<<1, 64>>>(it, d);
    commit_lat<<<1, 64>>>(it, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"err\": \"%s\", \"cluster_roundtrip_cycles\": {\"try_wait\": %llu, \"test_wait\": %llu, \"try_wait_hint20\": %llu}, "
           "\"cta_roundtrip_cycles\": {\"try_wait\": %llu, \"test_wait\": %llu}, \"commit_wait_cycles\": %llu}\n",
           cudaGetErrorString(e), h[0], h[1], h[2], h[4], h[5], h[8]);
    return 0;
}
