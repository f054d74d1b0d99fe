// launch_overhead.cu -- per-launch device time of near-empty kernels with the APNN kernels'
// launch attributes (dev aid): CUDA graph of 200 back-to-back launches, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2106_12169_b200/csrc launch_overhead.cu -o lo
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace apnn::sm100;

template <int MODE>
__global__ void __launch_bounds__(704, 1) k_plain(int* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t holder;
    if (MODE >= 1 && threadIdx.x / 32 == 0) {
        tmem_alloc_dyn(&holder, 512);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (MODE == 2 && threadIdx.x < 128) {   // 128 threads x 1 KB of strided int4 stores (like the int32 epilogue)
        int4* o = reinterpret_cast<int4*>(out) + (size_t)blockIdx.x * 128 * 64 + threadIdx.x * 64;
        for (int i = 0; i < 64; i++) o[i] = make_int4(i, i, i, i);
    }
    if (MODE >= 1) {
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x / 32 == 0) { tc_fence_after(); tmem_dealloc(holder, 512); }
    }
    if (out == nullptr) smem[threadIdx.x] = 1;
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(704, 1) k_cluster(int* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t holder;
    if (threadIdx.x / 32 == 0) tmem_alloc2(&holder, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (threadIdx.x / 32 == 0) { tc_fence_after(); tmem_dealloc2(holder, 512); }
    if (out == nullptr) smem[threadIdx.x] = 1;
}


// PDL: setup (TMEM alloc, barriers) before griddepcontrol.wait; dependents released at entry
template <int MODE>
__global__ void __launch_bounds__(704, 1) k_pdl(int* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t holder;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (MODE >= 1 && threadIdx.x / 32 == 0) tmem_alloc_dyn(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (MODE == 2 && threadIdx.x < 128) {
        int4* o = reinterpret_cast<int4*>(out) + (size_t)blockIdx.x * 128 * 64 + threadIdx.x * 64;
        for (int i = 0; i < 64; i++) o[i] = make_int4(i, i, i, i);
    }
    if (MODE >= 1) {
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x / 32 == 0) { tc_fence_after(); tmem_dealloc(holder, 512); }
    }
    if (out == nullptr) smem[threadIdx.x] = 1;
}

template <int MODE>
static void launch_pdl(int grid, int smem, cudaStream_t s, int* out) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(704);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_pdl<MODE>, out);
}

template <typename F>
static float graph_us(F launch) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    launch(s);
    cudaError_t e0 = cudaStreamSynchronize(s);
    cudaError_t el = cudaGetLastError();
    if (e0 != cudaSuccess || el != cudaSuccess) { printf("[launch error %s / %s]\n", cudaGetErrorString(e0), cudaGetErrorString(el)); return -1.f; }
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 200; i++) launch(s);
    cudaError_t e1 = cudaStreamEndCapture(s, &g);
    cudaError_t e2 = cudaGraphInstantiate(&ge, g, 0);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        printf("[graph error %s / %s]\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
        cudaGetLastError();
        return -1.f;
    }
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / 200;
}

int main() {
    int* out;
    cudaMalloc(&out, 148 * 128 * 1024 * 4);
    cudaGetLastError();
    const int SM = 225 * 1024;
    cudaFuncSetAttribute(k_plain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    cudaFuncSetAttribute(k_plain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    cudaFuncSetAttribute(k_plain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    cudaFuncSetAttribute(k_cluster<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    cudaFuncSetAttribute(k_pdl<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    cudaFuncSetAttribute(k_pdl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    for (int grid : {4, 32, 148}) {
        printf("grid %3d  plain 0smem %.2f us | plain 227K %.2f | +tmem %.2f | +tmem+strided 128KB stores %.2f | cluster2+tmem2 %.2f\n",
               grid, graph_us([&](cudaStream_t s) { k_plain<0><<<grid, 704, 0, s>>>(out); }),
               graph_us([&](cudaStream_t s) { k_plain<0><<<grid, 704, SM, s>>>(out); }),
               graph_us([&](cudaStream_t s) { k_plain<1><<<grid, 704, SM, s>>>(out); }),
               graph_us([&](cudaStream_t s) { k_plain<2><<<grid, 704, SM, s>>>(out); }),
               graph_us([&](cudaStream_t s) { k_cluster<0><<<grid, 704, SM, s>>>(out); }));
    }
    for (int grid : {4, 32, 148}) {
        printf("grid %3d  PDL: +tmem %.2f us | +tmem+stores %.2f | (no PDL, 8KB smem: %.2f)\n", grid,
               graph_us([&](cudaStream_t s) { launch_pdl<1>(grid, SM, s, out); }),
               graph_us([&](cudaStream_t s) { launch_pdl<2>(grid, SM, s, out); }),
               graph_us([&](cudaStream_t s) { k_plain<1><<<grid, 704, 8192, s>>>(out); }));
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
