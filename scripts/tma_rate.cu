// tma_rate.cu -- TMA load issue/complete rate for the box shapes the APNN kernels use (dev aid).
// One CTA per SM, one thread issues `iters` TMA loads into an 8-deep smem ring (mbarrier
// complete_tx, no consumers); reports clocks per box and bytes/clock/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2106_12169_b200/csrc tma_rate.cu -o tma_rate -lcuda
#include <cuda.h>
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace apnn::sm100;

__host__ __device__ inline int depth_of(int box_bytes) {
    int d = 200 * 1024 / box_bytes;
    return d > 64 ? 64 : d;
}

template <int DIMS>
__global__ void __launch_bounds__(32, 1) rate_kernel(const __grid_constant__ CUtensorMap tm, int iters, int box_bytes,
                                                     int c1_span, int c1_step, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[64];
    const int D = depth_of(box_bytes);
    if (threadIdx.x != 0) return;
    tma_prefetch(&tm);
    for (int i = 0; i < D; i++) mbar_init(&bars[i], 1);
    fence_mbar_init();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const int s = it % D;
        if (it >= D) mbar_wait(&bars[s], ((it / D) - 1) & 1);
        mbar_arrive_expect_tx(&bars[s], box_bytes);
        const int c1 = ((it * c1_step) + blockIdx.x * 131) % c1_span;
        uint8_t* dst = smem + s * box_bytes;
        if (DIMS == 3) {  // 4 boxes of box_bytes/4 per barrier (2-D map, rows c1..)
            for (int g = 0; g < 4; g++)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             :: "r"(smem_u32(dst + g * (box_bytes / 4))), "l"(&tm), "r"(smem_u32(&bars[s])), "r"(0), "r"(c1 + g * 32) : "memory");
        } else if (DIMS == 2) asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                    :: "r"(smem_u32(dst)), "l"(&tm), "r"(smem_u32(&bars[s])), "r"(0), "r"(c1) : "memory");
        else if (DIMS == 4) tma_load_4d(dst, &tm, &bars[s], 0, c1, 0, 0);
        else tma_load_5d(dst, &tm, &bars[s], 0, c1 % 200 - 1, 0, c1 / 200 % 200, 0);
    }
    for (int it = iters - D; it < iters; it++) mbar_wait(&bars[it % D], (it / D) & 1);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
}

// L lanes of one warp each own every L-th ring stage: one warp instruction issues L
// expect_tx arrivals and L boxes (2-D map)
template <int L>
__global__ void __launch_bounds__(32, 1) lanes_kernel(const __grid_constant__ CUtensorMap tm, int iters, int box_bytes,
                                                      int c1_span, int c1_step, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[64];
    const int D = depth_of(box_bytes) / L * L;
    const int lane = threadIdx.x;
    if (lane == 0) {
        tma_prefetch(&tm);
        for (int i = 0; i < D; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane >= L) return;
    unsigned long long t0 = clock64();
    for (int it = lane; it < iters; it += L) {
        const int s = it % D;
        if (it >= D) mbar_wait(&bars[s], ((it / D) - 1) & 1);
        mbar_arrive_expect_tx(&bars[s], box_bytes);
        const int c1 = ((it * c1_step) + blockIdx.x * 131) % c1_span;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     :: "r"(smem_u32(smem + s * box_bytes)), "l"(&tm), "r"(smem_u32(&bars[s])), "r"(0), "r"(c1) : "memory");
    }
    for (int it = iters - D + lane; it < iters; it += L) mbar_wait(&bars[it % D], (it / D) & 1);
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    Enc enc = (Enc)fnp;
    void* buf;
    const size_t bytes = 256ull << 20;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    unsigned long long* dout;
    cudaMalloc(&dout, 148 * 8);
    const int iters = 4000, sms = 148;
    auto run = [&](const char* name, int dims, CUtensorMap& tm, int box_bytes, int span, int step) {
        void (*k)(CUtensorMap, int, int, int, int, unsigned long long*) =
            dims == 2 ? rate_kernel<2> : (dims == 3 ? rate_kernel<3> : (dims == 4 ? rate_kernel<4> : rate_kernel<5>));
        const int smem = depth_of(box_bytes) * box_bytes;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<sms, 32, smem>>>(tm, iters, box_bytes, span, step, dout);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; i++) avg += h[i];
        avg /= sms;
        printf("%-48s depth %2d box %6d B: %7.1f clk/box  %6.1f B/clk/SM  (%s)\n", name, depth_of(box_bytes), box_bytes, avg / iters,
               box_bytes * iters / avg, cudaGetErrorString(e));
        (void)0;
    };
    CUtensorMap tm;
    cuuint32_t e1[5] = {1, 1, 1, 1, 1};
    {   // GEMM A: packed [rows][2 planes][256 words] (K = 8192), box {4 words, 128 rows, 2 planes}
        cuuint64_t d[4] = {256, 65536, 2, 1}, st[3] = {2 * 256 * 4, 256 * 4, 2 * 256 * 4 * 65536ull};
        cuuint32_t b[4] = {4, 128, 2, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("gemm A {4w,128 rows,2 planes} (16-B lines)", 4, tm, 4096, 65536 - 128, 128);
    }
    {   // GEMM B: 1 plane, 128 rows
        cuuint64_t d[4] = {256, 65536, 1, 1}, st[3] = {256 * 4, 256 * 4, 256 * 4 * 65536ull};
        cuuint32_t b[4] = {4, 128, 1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("gemm B {4w,128 rows,1 plane} (16-B lines)", 4, tm, 2048, 65536 - 128, 128);
    }
    {   // conv act: {Cw=4, W=200, bits=2, H=200, B=1}, box {4, 28 px, 2, 1, 1}
        cuuint64_t d[5] = {4, 200, 2, 200, 1};
        cuuint64_t st[4] = {32, 16, 32 * 200, 32 * 200 * 200};
        cuuint32_t b[5] = {4, 28, 2, 1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("conv act 5-D {4w,28 px,2 planes,1,1}", 5, tm, 28 * 32, 40000, 201);
    }
    {   // same data as {8 words (both planes), 28 px}: 32-B lines
        cuuint64_t d[2] = {8, 40000}, st[1] = {32};
        cuuint32_t b[2] = {8, 28};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("conv act 2-D {8w (2 planes),28 px} (32-B lines)", 2, tm, 28 * 32, 40000 - 28, 201);
    }
    {   // 2-D {16 words, 128 rows}: 64-B lines
        cuuint64_t d[2] = {256, 65536}, st[1] = {1024};
        cuuint32_t b[2] = {16, 128};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("2-D {16w,128 rows} (64-B lines)", 2, tm, 8192, 65536 - 128, 128);
    }
    {   // 2-D {32 words, 128 rows}: 128-B lines
        cuuint64_t d[2] = {256, 65536}, st[1] = {1024};
        cuuint32_t b[2] = {32, 128};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("2-D {32w,128 rows} (128-B lines)", 2, tm, 16384, 65536 - 128, 128);
    }
    {   // 4 boxes {32w, 32 rows} per barrier
        cuuint64_t d[2] = {256, 65536}, st[1] = {1024};
        cuuint32_t b[2] = {32, 32};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("4 x 2-D {32w,32 rows} per barrier (per 4 boxes)", 3, tm, 16384, 65536 - 256, 128);
    }
    {   // 4 boxes {4w, 32 rows} per barrier: small 16-B-line boxes
        cuuint64_t d[2] = {256, 65536}, st[1] = {1024};
        cuuint32_t b[2] = {4, 32};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("4 x 2-D {4w,32 rows} per barrier (per 4 boxes)", 3, tm, 2048, 65536 - 256, 128);
    }
    for (int L : {1, 2, 4, 8}) {
        cuuint64_t d[2] = {256, 65536}, st[1] = {1024};
        cuuint32_t b[2] = {4, 128};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, d, st, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        void (*k)(CUtensorMap, int, int, int, int, unsigned long long*) =
            L == 1 ? lanes_kernel<1> : L == 2 ? lanes_kernel<2> : L == 4 ? lanes_kernel<4> : lanes_kernel<8>;
        const int box = 2048, smem = depth_of(box) * box;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<sms, 32, smem>>>(tm, iters, box, 65536 - 256, 128, dout);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; i++) avg += h[i];
        avg /= sms;
        printf("%d lanes issuing {4w,128 rows} boxes, own barriers: %7.1f clk/box (%s)\n", L, avg / iters, cudaGetErrorString(e));
    }
    return 0;
}
