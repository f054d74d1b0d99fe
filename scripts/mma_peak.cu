// mma_peak.cu -- microbenchmark of tcgen05.mma kind::i8 issue rate on B200 (sm_100a).
// Measures the int8 tensor-core ceiling for the instruction shapes the APNN kernels use:
//   mode 0: 1-CTA  M=128 N=256 K=32, A smem  (SS)
//   mode 1: 1-CTA  M=128 N=256 K=32, A TMEM  (TS)
//   mode 2: 2-CTA  M=256 N=256 K=32, A smem  (SS, cta_group::2)
//   mode 3: 2-CTA  M=256 N=256 K=32, A TMEM  (TS, cta_group::2)
//   mode 4: 1-CTA  M=128 N=256 K=64, kind::mxf4 block32 (e2m1, E8M0 scales in TMEM), SS
//   mode 5: 2-CTA  M=256 N=256 K=64, kind::mxf4 block32, SS (cta_group::2)
//   mode 6 / 7: 2-CTA M=256 N=64 / 128 K=32, kind::i8, A smem (SS): issue rate at small N
//   mode 8 / 10: 2-CTA M=256 N=224 / 128 K=64, kind::mxf4 (tile widths of the fp4 pair kernels)
//   mode 9: as mode 5 with a multicast tcgen05.commit after every 4 MMAs (the kernels' per-stage commit)
//   mode 11: as mode 9 with A/B cycling over 6 stages of a 192 KB ring (the pair kernel's operand addresses)
//   mode 12: as mode 11 with the 6 stages' operands filled with random bytes (data-dependent power / clock)
// Operands are zeros (timing is value-independent).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2106_12169_b200/csrc mma_peak.cu -o mma_peak
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace apnn::sm100;

template <int MODE>
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;            // 128 rows x 128 B (one K=128 block)
    uint8_t* sB = smem + 16384;    // 256 rows x 128 B (1-CTA) / 128 rows (2-CTA)
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    constexpr bool two = MODE == 2 || MODE == 3 || MODE == 5 || MODE >= 6;
    constexpr bool fp4 = MODE == 4 || MODE == 5 || MODE >= 8;
    constexpr bool ring = MODE == 11 || MODE == 12;
    constexpr int NN = MODE == 6 ? 64 : (MODE == 7 || MODE == 10 ? 128 : (MODE == 8 ? 224 : 256));
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < (ring ? 6 * 32768 : 49152) / 16; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
        reinterpret_cast<uint4*>(smem)[i] = MODE == 12 ? make_uint4(h, h * 3u + 1u, h ^ 0x9E3779B9u, h * 7u) : make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();
    if (warp == 0) {
        if (two) tmem_alloc2(&holder, 512); else tmem_alloc_dyn(&holder, 512);
    }
    tc_fence_before();
    __syncthreads();
    if (two) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = holder;
    const bool leader = !two || cluster_ctarank() == 0;
    __shared__ uint64_t cbar;
    if ((MODE == 9 || ring) && threadIdx.x == 0) { mbar_init(&cbar, 1); fence_mbar_init(); }
    if (fp4) {  // scale-factor columns 256..287 of every lane: E8M0 127 (2^0)
        const uint32_t ones[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
        const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
        for (uint32_t c = 0; c < 32; c += 8) tmem_st8(lb + 256 + c, ones);
        tmem_wait_st();
        tc_fence_before();
        __syncthreads();
        if (two) cluster_sync();
        tc_fence_after();
    }
    unsigned long long t0 = clock64();
    if (warp == 1 && leader && (threadIdx.x % 32) == 0) {
        const uint32_t idesc = idesc_i8(two ? 256 : 128, NN, false, false);
        const uint32_t abase = smem_u32(sA), bbase = smem_u32(sB);
        for (int it = 0; it < iters; it++) {
            const uint32_t sa = ring ? abase + (uint32_t)(it % 6) * 32768u : abase;
            const uint32_t sbb = ring ? abase + (uint32_t)(it % 6) * 32768u + 16384u : bbase;
#pragma unroll
            for (int kk = 0; kk < 4; kk++) {
                const uint64_t bd = umma_desc_sw128(sbb + kk * 32, 1024);
                if (MODE == 0) mma_i8_ss(tmem, umma_desc_sw128(abase + kk * 32, 1024), bd, idesc, 1);
                if (MODE == 1) mma_i8_ts(tmem, tmem + 256 + kk * 8, bd, idesc, 1);
                if (MODE == 2 || MODE == 6 || MODE == 7) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(umma_desc_sw128(abase + kk * 32, 1024)), "l"(bd), "r"(idesc) : "memory");
                }
                if (MODE == 3) mma2_i8_ts(tmem, tmem + 256 + kk * 8, bd, idesc, 1);
                if (fp4) {
                    const uint32_t id4 = (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | (1u << 23) |
                                         ((uint32_t)((MODE != 4 ? 256 : 128) >> 4) << 24);
                    if (MODE == 4)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
                                     ::"r"(tmem), "l"(umma_desc_sw128(abase + kk * 32, 1024)), "l"(bd), "r"(id4),
                                     "r"(tmem + 256), "r"(tmem + 272) : "memory");
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
                                     ::"r"(tmem), "l"(umma_desc_sw128(sa + kk * 32, 1024)), "l"(bd), "r"(id4),
                                     "r"(tmem + 256), "r"(tmem + 272) : "memory");
                }
            }
            if (MODE == 9 || ring) mma2_commit_mc(&cbar, 0x3);
        }
        if (two) mma2_commit_mc(&bar, 0x3); else mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (two) cluster_sync();
    if (warp == 0) { tc_fence_after(); if (two) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(int iters, int sms) {
    auto k = peak_kernel<MODE>;
    const int smem_bytes = (MODE == 11 || MODE == 12) ? 6 * 32768 + 1024 : 49152 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    unsigned long long* d;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    constexpr bool two = MODE == 2 || MODE == 3 || MODE == 5 || MODE >= 6;
    (void)two;
    attr[0].val.clusterDim.x = two ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k, iters / 10, d);  // warm-up
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, iters, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc[512];
    cudaMemcpy(cyc, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    const double M = two ? 256 : 128;
    const double Kst = (MODE == 4 || MODE == 5 || MODE >= 8) ? 64 : 32;
    const double NN = MODE == 6 ? 64 : (MODE == 7 || MODE == 10 ? 128 : (MODE == 8 ? 224 : 256));  // K per instruction (fp4: 64 elements in 32 bytes)
    const int units = two ? sms / 2 : sms;
    const double ops = 2.0 * M * NN * Kst * 4.0 * iters * units;
    printf("{\"mode\": %d, \"name\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f, \"cycles_cta0\": %llu, "
           "\"mac_per_clk_per_sm\": %.0f, \"clk_ghz_cta0\": %.3f}\n",
           MODE, MODE == 0 ? "i8_1cta_SS" : MODE == 1 ? "i8_1cta_TS" : MODE == 2 ? "i8_2cta_SS" : MODE == 3 ? "i8_2cta_TS"
                 : MODE == 4 ? "mxf4_1cta_SS" : MODE == 5 ? "mxf4_2cta_SS" : MODE == 6 ? "i8_2cta_SS_N64" : MODE == 7 ? "i8_2cta_SS_N128"
                 : MODE == 8 ? "mxf4_2cta_N224" : MODE == 9 ? "mxf4_2cta_commit_per_4" : MODE == 10 ? "mxf4_2cta_N128"
                 : MODE == 11 ? "mxf4_2cta_ring6" : "mxf4_2cta_ring6_random",
           cudaGetErrorString(err), ms, ops / (ms * 1e-3) / 1e12, cyc[0],
           (M * NN * Kst * 4.0 * iters) / (double)cyc[0] / (two ? 2 : 1), (double)cyc[0] / (ms * 1e6));
    cudaFree(d);
}

int main(int argc, char** argv) {
    int iters = argc > 1 ? atoi(argv[1]) : 20000;
    int sms = 148;
    run<0>(iters, sms);
    run<1>(iters, sms);
    run<2>(iters, sms);
    run<3>(iters, sms);
    run<4>(iters, sms);
    run<5>(iters, sms);
    run<6>(iters, sms);
    run<7>(iters, sms);
    run<8>(iters, sms);
    run<9>(iters, sms);
    run<10>(iters, sms);
    run<11>(iters, sms);
    run<12>(iters, sms);
    return 0;
}
