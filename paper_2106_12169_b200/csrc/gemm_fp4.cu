// gemm_fp4.cu -- exact FP4 formulation of the AP-bit contraction (row f3, APNN_VARIANT_TC_FP4).
//
// For operands of at most 2 bits (0/1 codes 0..3, or +-1), every value is exactly
// representable in e2m1 (0, 1, 2, 3 = 0x0, 0x2, 0x4, 0x5; +-1 = 0x2 / 0xA), every product
// is an integer of magnitude <= 9, and an fp32 accumulator is exact while |Y| < 2^24
// (host check K * max|a| * max|w| < 2^24).  So the bit combination of PAPER.md:1426-1429,
// applied to the operands as in the int8 path, can feed
// `tcgen05.mma kind::mxf4.block_scale` with all block scales 2^0 (E8M0 127): the fp4 pipe,
// twice the int8 rate on B200, and half the operand bytes the recombination writes.
//
// Kernel (one CTA, 128 x BN output tile, BN = 128 or 256):
//   warp 0      TMA producer: planes of 2 k-blocks (256 K elements) per stage
//   warp 1      TMEM allocator, single-thread MMA issuer (4 x 128xBNx64 per stage)
//   warps 2-9   recombination planes -> e2m1 nibbles into the K-major SWIZZLE_128B operand
//               tiles (A and B both in shared memory), then the epilogue (fp32 -> int32,
//               int32 store or the fused requantisation of tc_common.cuh)
// Element order: 16-byte chunk (kb2*4 + gi) of a row holds the 32 elements of group gi of
// k-block kb2; word j of it holds elements {j, j+4, ..., j+28} (nibble n = element j+4n):
// the same permutation for A and B, so the dot product is unchanged.
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "tc_common.cuh"

namespace apnn {
namespace fp4 {

using namespace sm100;

constexpr int BM = 128;
constexpr int THREADS = 10 * 32;
constexpr int MAXS = 6;    // operand stages
constexpr int MAXSP = 12;  // packed-plane stages (a deeper ring: TMA latency)
constexpr uint32_t kSfCols = 16;  // scale-factor TMEM columns per operand (all bytes 0x7F = 2^0)

struct Params {
    Geom g;
    Epi e;
    void* Y;
    int stages;
    int pstages;
    int nst;             // stages (of 2 k-blocks) along K
    uint32_t a_bytes;    // plane bytes per stage (A: 128 rows x a_bits x 32 B)
    uint32_t b_bytes;    // (B: BN rows x w_bits x 32 B)
    uint32_t tmem_cols;
    int tab_mode;
};

// block-scaled instruction descriptor: E2M1 x E2M1 (MXF4 format 1), fp32 D, K-major,
// E8M0 scales, M = 128, N, dense K = 64 (cute::UMMA::InstrDescriptorBlockScaled layout)
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7)                      // A format: E2M1
           | (1u << 10)                   // B format: E2M1
           | ((uint32_t)(N >> 3) << 17)   // N / 8
           | (1u << 23)                   // scale format: E8M0
           | ((uint32_t)(M >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void mma_mxf4(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
            d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_sw(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// 32 elements of one plane group -> 4 words of e2m1 nibbles (word j: elements j + 4n)
template <int NB, bool PM1>
__device__ __forceinline__ void decode_group_fp4(const uint32_t (&pw)[2], uint32_t vm, bool masked,
                                                 uint32_t (&o)[4]) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint32_t b0 = (pw[0] >> j) & 0x11111111u;
        uint32_t w;
        if (PM1) {  // +1 -> 0x2, -1 -> 0xA; elements outside vm -> 0
            w = 0x22222222u | ((b0 ^ 0x11111111u) << 3);
            if (masked) w &= ((vm >> j) & 0x11111111u) * 0xFu;
        } else if (NB == 1) {  // 0 -> 0x0, 1 -> 0x2
            w = b0 << 1;
        } else {  // 0, 1, 2, 3 -> 0x0, 0x2, 0x4, 0x5
            const uint32_t b1 = (pw[1] >> j) & 0x11111111u;
            w = (b1 << 2) | ((b0 & ~b1) << 1) | (b0 & b1);
        }
        o[j] = w;
    }
}

// one operand row of a stage (2 k-blocks): planes smem [plane][rows][32 B] -> 128-byte
// K-major SWIZZLE_128B row of e2m1 nibbles
template <int NB, bool PM1>
__device__ __forceinline__ void recomb_row(const uint8_t* planes, int rows, int row, uint8_t* op, int kvalid0) {
    const uint4* src = reinterpret_cast<const uint4*>(planes);
    uint4 v[NB][2];
#pragma unroll
    for (int pl = 0; pl < NB; pl++) {
        v[pl][0] = src[(pl * rows + row) * 2];
        v[pl][1] = src[(pl * rows + row) * 2 + 1];
    }
#pragma unroll
    for (int kb2 = 0; kb2 < 2; kb2++) {
        const int kvalid = kvalid0 - kb2 * 128;
#pragma unroll
        for (int gi = 0; gi < 4; gi++) {
            uint32_t pw[2] = {0u, 0u};
#pragma unroll
            for (int pl = 0; pl < NB; pl++) pw[pl] = tc::sel4(v[pl][kb2], gi);
            uint32_t o[4];
            decode_group_fp4<NB, PM1>(pw, tc::valid_mask(kvalid, gi), PM1 && kvalid < 128, o);
            *reinterpret_cast<uint4*>(op + tc::b_chunk_offset(row, kb2 * 4 + gi)) = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

// apnn_prepare_weights: packed W [N][w_bits][Kw] -> e2m1 [N][Kw*16 bytes]; 16 bytes per
// 32-element group g at byte 16*g (the kernel's chunk order), elements >= K are value 0.
template <int NB, bool PM1>
__global__ void __launch_bounds__(256) prepare_kernel(const uint32_t* __restrict__ W, int N, int K, int Kw,
                                                      uint8_t* __restrict__ out) {
    // a thread takes 4 consecutive groups (one 16-byte word of each plane, Kw is a multiple of 4):
    // 32-bit index math only (the 64-bit division of a flat index was the kernel's cost)
    const int Kq = Kw / 4;
    for (int n = blockIdx.y * blockDim.y + threadIdx.y; n < N; n += gridDim.y * blockDim.y) {
        const uint32_t* wrow = W + (long long)n * NB * Kw;
        uint8_t* orow = out + (long long)n * Kw * 16;
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Kq; q += gridDim.x * blockDim.x) {
            uint4 pv[2];
#pragma unroll
            for (int pl = 0; pl < NB; pl++) pv[pl] = __ldg(reinterpret_cast<const uint4*>(wrow + (long long)pl * Kw) + q);
            uint4 o4[4];
#pragma unroll
            for (int gi = 0; gi < 4; gi++) {
                const int gidx = q * 4 + gi;
                uint32_t pw[2] = {0u, 0u};
#pragma unroll
                for (int pl = 0; pl < NB; pl++) pw[pl] = tc::sel4(pv[pl], gi);
                const int nv = K - gidx * 32;
                const uint32_t vm = nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
                uint32_t o[4];
                decode_group_fp4<NB, PM1>(pw, vm, true, o);
                if (!PM1) {  // 0/1 codes: padding bits are zero already; mask anyway (robust to dirty padding)
#pragma unroll
                    for (int j = 0; j < 4; j++) o[j] &= ((vm >> j) & 0x11111111u) * 0xFu;
                }
                o4[gi] = make_uint4(o[0], o[1], o[2], o[3]);
            }
#pragma unroll
            for (int gi = 0; gi < 4; gi++) reinterpret_cast<uint4*>(orow)[q * 4 + gi] = o4[gi];
        }
    }
}

template <bool PM1>
__device__ __forceinline__ void recomb_row_any(int nb, const uint8_t* planes, int rows, int row, uint8_t* op,
                                               int kvalid) {
    if (PM1) recomb_row<1, true>(planes, rows, row, op, kvalid);
    else if (nb == 1) recomb_row<1, false>(planes, rows, row, op, kvalid);
    else recomb_row<2, false>(planes, rows, row, op, kvalid);
}

// one k-block (kb2 of the stage) of one A row (prepared-weights mode: the 8 recombination
// warps split the stage's two k-blocks)
template <int NB, bool PM1>
__device__ __forceinline__ void recomb_row_kb(const uint8_t* planes, int rows, int row, uint8_t* op, int kb2,
                                              int kvalid) {
    const uint4* src = reinterpret_cast<const uint4*>(planes);
    uint4 v[NB];
#pragma unroll
    for (int pl = 0; pl < NB; pl++) v[pl] = src[(pl * rows + row) * 2 + kb2];
#pragma unroll
    for (int gi = 0; gi < 4; gi++) {
        uint32_t pw[2] = {0u, 0u};
#pragma unroll
        for (int pl = 0; pl < NB; pl++) pw[pl] = tc::sel4(v[pl], gi);
        uint32_t o[4];
        decode_group_fp4<NB, PM1>(pw, tc::valid_mask(kvalid, gi), PM1 && kvalid < 128, o);
        *reinterpret_cast<uint4*>(op + tc::b_chunk_offset(row, kb2 * 4 + gi)) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// PREP: W arrives pre-recombined (apnn_prepare_weights: e2m1 nibbles in the kernel's element
// order, padding = value 0) and is loaded by TMA straight into the SWIZZLE_128B operand tile;
// only A is recombined per tile.
template <int BN, bool A_PM1, bool W_PM1, bool PREP = false, bool I32 = false>
__global__ void __launch_bounds__(THREADS, BN == 192 ? 2 : 1)  // BN = 192: two CTAs per SM (TMEM 256 cols each)
    fp4_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB, const Params p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages, SP = p.pstages;
    uint8_t* sAop = smem;                                   // S x 128 x 128 B
    uint8_t* sBop = sAop + (size_t)S * BM * 128;            // S x BN x 128 B
    uint8_t* sApl = sBop + (size_t)S * BN * 128;            // SP x a_bytes
    uint8_t* sBpl = sApl + (size_t)SP * p.a_bytes;          // SP x b_bytes
    int32_t* sTab = reinterpret_cast<int32_t*>(sBpl + (size_t)SP * p.b_bytes);  // BN x kTabStride
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + BN * tc::kTabStride);
    uint64_t* plane_full = bars;                            // [MAXSP]
    uint64_t* plane_empty = bars + MAXSP;                   // [MAXSP]
    uint64_t* op_full = bars + 2 * MAXSP;                   // [MAXS]
    uint64_t* op_empty = op_full + MAXS;                    // [MAXS]
    uint64_t* accum_full = op_empty + MAXS;
    uint64_t* b_full = accum_full + 2;                      // [MAXS] (PREP: B operand landed)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(b_full + MAXS);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const Geom& g = p.g;
    const int nst = p.nst;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmapA);
        tma_prefetch(&tmapB);
        for (int s = 0; s < SP; s++) {
            mbar_init(&plane_full[s], 1);
            mbar_init(&plane_empty[s], 8);
        }
        for (int s = 0; s < S; s++) {
            mbar_init(&op_full[s], 8);
            mbar_init(&op_empty[s], 1);
            mbar_init(&b_full[s], 1);
        }
        mbar_init(accum_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_dyn(tmem_holder, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const uint32_t sfa = tmem + BN, sfb = tmem + BN + kSfCols;
    if (warp >= 2 && warp < 6) {  // every scale factor byte = E8M0 127 (2^0), all 128 lanes
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // warp w owns lanes 32*(w%4)..
        const uint32_t ones[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
#pragma unroll
        for (uint32_t c = 0; c < 2 * kSfCols; c += 8) tmem_st8(lane_base + BN + c, ones);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            int os = 0;
            uint32_t oph = 0;
            for (int i = 0; i < nst; i++, s = (s + 1 == SP) ? 0 : s + 1, ph ^= (s == 0),
                     os = (os + 1 == S) ? 0 : os + 1, oph ^= (os == 0)) {  // no divisions
                mbar_wait(&plane_empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&plane_full[s], p.a_bytes + (PREP ? 0u : p.b_bytes));
                tma_load_4d(sApl + (size_t)s * p.a_bytes, &tmapA, &plane_full[s], i * 8, m0, 0, 0);
                if (!PREP) {
                    tma_load_4d(sBpl + (size_t)s * p.b_bytes, &tmapB, &plane_full[s], i * 8, n0, 0, 0);
                } else {  // prepared W: 128 bytes (256 e2m1) x BN rows straight into operand stage os
                    mbar_wait(&op_empty[os], oph ^ 1);
                    mbar_arrive_expect_tx(&b_full[os], (uint32_t)BN * 128);
                    tma_load_2d_sw(sBop + (size_t)os * BN * 128, &tmapB, &b_full[os], i * 128, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = idesc_mxf4(BM, BN);
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nst; i++, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0)) {
                mbar_wait(&op_full[s], ph);
                if (PREP) mbar_wait(&b_full[s], ph);
                tc_fence_after();
                const uint32_t abase = smem_u32(sAop + (size_t)s * BM * 128);
                const uint32_t bbase = smem_u32(sBop + (size_t)s * BN * 128);
#pragma unroll
                for (int kk = 0; kk < 4; kk++)  // K = 64 fp4 elements = 32 bytes per MMA
                    mma_mxf4(tmem, tc::b_desc(abase, kk), tc::b_desc(bbase, kk), idesc, sfa, sfb, (i | kk) != 0);
                mma_commit(&op_empty[s]);
            }
            mma_commit(accum_full);
        }
    } else {
        const int q = warp & 3;
        const int grp = (warp - 2) >> 2;  // 0: A rows, 1: B rows (BN = 128) / B rows t, t+128
        const int t = q * 32 + lane;
        const int et = threadIdx.x - 64;
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        if ((p.tab_mode == tc::kTabQ3 || p.tab_mode == tc::kTabHybrid) && et < BN)
            tc::build_threshold_row(sTab + et * tc::kTabStride, n0 + et, g.N, p.e);
        int s = 0, ps = 0;
        uint32_t ph = 0, pph = 0;
        for (int i = 0; i < nst; i++, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0),
                 ps = (ps + 1 == SP) ? 0 : ps + 1, pph ^= (ps == 0)) {
            int kvalid = 256;  // +-1 x +-1: padded K decodes to 0
            if (A_PM1 && W_PM1) {
                const int rem = g.K - i * 256;
                kvalid = rem < 256 ? rem : 256;
            }
            mbar_wait(&plane_full[ps], pph);
            mbar_wait(&op_empty[s], ph ^ 1);
            if (PREP) {  // prepared W has value-0 padding: A needs no mask; grp = k-block of the stage
                const uint8_t* apl = sApl + (size_t)ps * p.a_bytes;
                uint8_t* aop = sAop + (size_t)s * BM * 128;
                if (A_PM1) recomb_row_kb<1, true>(apl, BM, t, aop, grp, 128);
                else if (g.a_bits == 1) recomb_row_kb<1, false>(apl, BM, t, aop, grp, 128);
                else recomb_row_kb<2, false>(apl, BM, t, aop, grp, 128);
            } else if (grp == 0) {
                recomb_row_any<A_PM1>(g.a_bits, sApl + (size_t)ps * p.a_bytes, BM, t, sAop + (size_t)s * BM * 128,
                                      kvalid);
            } else {
                const uint8_t* bpl = sBpl + (size_t)ps * p.b_bytes;
                uint8_t* bop = sBop + (size_t)s * BN * 128;
                recomb_row_any<W_PM1>(g.w_bits, bpl, BN, t, bop, kvalid);
                if (BN > 128 && t + 128 < BN) recomb_row_any<W_PM1>(g.w_bits, bpl, BN, t + 128, bop, kvalid);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&plane_empty[ps]);
                mbar_arrive(&op_full[s]);
            }
        }
        named_bar_sync(1, 256);  // threshold table complete
        mbar_wait(accum_full, 0);
        tc_fence_after();
        const int m = m0 + t;
        constexpr int half = BN / 2;
        // int32 output: stage each 32 x 32 block in the (now idle) operand smem and write it back
        // coalesced (4 full 128-byte row segments per store instruction) instead of one row per lane
        // (compile-time: the branch in the fused instances cost them ~6 % -- register allocation)
        constexpr bool lsu = I32;
        uint8_t* stg = smem + (warp - 2) * 4096;
#pragma unroll 1
        for (int c = grp * half; c < (grp + 1) * half; c += 32) {
            uint32_t acc[32];
            tmem_ld32(tmem_lane + c, acc);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; k++) acc[k] = (uint32_t)__float2int_rn(__uint_as_float(acc[k]));  // exact
            if (lsu) {
                tc::stage_int32_chunk(acc, stg, lane);
                __syncwarp();
                tc::writeback_int32_block(stg, lane, reinterpret_cast<int32_t*>(p.Y), m0 + q * 32, g.M, n0 + c, g.N);
                __syncwarp();
                continue;
            }
            tc::epilogue_chunk(acc, m, n0 + c, c, g, p.e, p.Y, sTab, p.tab_mode);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, p.tmem_cols);
    }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
        else
            cudaGetLastError();
    });
    return fn;
}

// packed [rows][bits][Kw] as {Kw, rows, bits}; box {8 words = 2 k-blocks, box_rows, bits}
// lands as [plane][row][32 B]
bool make_map(CUtensorMap* m, const uint32_t* base, int rows, int bits, int Kw, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)Kw, (cuuint64_t)rows, (cuuint64_t)bits, 1};
    cuuint64_t strides[3] = {(cuuint64_t)bits * Kw * 4, (cuuint64_t)Kw * 4, (cuuint64_t)bits * Kw * 4 * rows};
    cuuint32_t box[4] = {8, (cuuint32_t)box_rows, (cuuint32_t)bits, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// prepared W [N][Kw*16 bytes] as a 2-D byte tensor; box {128 bytes, BN rows} with
// SWIZZLE_128B lands exactly in the UMMA K-major SWIZZLE_128B operand layout
bool make_map_prep(CUtensorMap* m, const uint8_t* base, int N, int Kw, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)Kw * 16, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)Kw * 16};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// operand rows of row_bytes bytes (prepared e2m1 or int8); box {128 bytes, box_rows}, SWIZZLE_128B
bool make_map_rows(CUtensorMap* m, const uint8_t* base, int rows, int row_bytes, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool AP, bool WP, bool PREP>
static cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, dim3 grid, size_t smem,
                          cudaStream_t s) {
    auto kfn = (p.e.out_bits == 0 && (p.g.N & 3) == 0) ? fp4_kernel<BN, AP, WP, PREP, true>
                                                        : fp4_kernel<BN, AP, WP, PREP, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    kfn<<<grid, THREADS, smem, s>>>(ta, tb, p);
    return cudaGetLastError();
}

template <int BN, bool PREP>
static cudaError_t launch_enc(int enc, const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, dim3 grid,
                              size_t smem, cudaStream_t s) {
    switch (enc) {
    case APNN_ENC_01_01: return launch<BN, false, false, PREP>(ta, tb, p, grid, smem, s);
    case APNN_ENC_PM1_PM1: return launch<BN, true, true, PREP>(ta, tb, p, grid, smem, s);
    case APNN_ENC_W_PM1_A_01: return launch<BN, false, true, PREP>(ta, tb, p, grid, smem, s);
    default: return launch<BN, true, false, PREP>(ta, tb, p, grid, smem, s);
    }
}

}  // namespace fp4

static bool fp4_dual() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_FP4_BN192");
        v = s ? atoi(s) : 0;  // experiment: +4.7 % in the CUDA-graph sweep, -1..2 % in the bench (L2 flushed;
                              // ncu 376.5 vs 350.8 us: the A decode per MAC grows by 256/192)
    }
    return v != 0;
}

static int fp4_op_stages() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_FP4_S");
        v = s ? atoi(s) : 3;  // measured (8192^3 w1a2 fused): S = 2 / 3 / 4 -> 2616 / 2922 / 2926 TOPS
        if (v < 2) v = 2;
        if (v > fp4::MAXS) v = fp4::MAXS;
    }
    return v;
}

// GEMM with both operands of at most 2 bits and |Y| < 2^24 (exact fp32 accumulation)
bool tc_fp4_supports(const Geom& g) {
    if (g.conv || g.K <= 0 || g.M <= 0 || g.N <= 0 || g.a_bits > 2 || g.w_bits > 2) return false;
    const long long ma = (g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_01_A_PM1) ? 1 : (1 << g.a_bits) - 1;
    const long long mw = (g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_PM1_A_01) ? 1 : (1 << g.w_bits) - 1;
    return (long long)g.K * ma * mw < (1LL << 24);
}

static cudaError_t launch_fp4_impl(const uint32_t* A, const void* W, bool prep, const Geom& g, const Epi& e,
                                   void* Y, cudaStream_t s) {
    using namespace fp4;
    Params p;
    std::memset(&p, 0, sizeof(p));
    p.g = g;
    p.e = e;
    p.Y = Y;
    const int Kw = (g.K + 127) / 128 * 4;
    p.nst = (Kw + 7) / 8;  // stages of 2 k-blocks (the TMA zero-fills a missing second k-block)
    p.tab_mode = tc::kTabNone;
    if (e.out_bits > 0 && e.out_bits <= 2) p.tab_mode = tc::kTabQ3;
    else if (e.out_bits > 2 && (unsigned long long)e.qmax * (unsigned long long)e.S <= 0xFFFFFFFFull)
        p.tab_mode = tc::kTabHybrid;
    const int ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;
    // prepared W, fused output: 128 x 192 tiles, two CTAs per SM (one's epilogue overlaps the
    // other's main loop; TMEM 192 + 32 scale columns -> 256 each); experiment knob APNN_FP4_BN192=1
    const bool dual = prep && g.N > 128 && e.out_bits > 0 && fp4_dual();  // measured: +3-5 % fused, int32 even
    const int BN = dual ? 192 : (g.N > 128 ? 256 : 128);
    p.a_bytes = 32u * BM * g.a_bits;
    p.b_bytes = prep ? 0u : 32u * BN * g.w_bits;
    const size_t op = (size_t)(BM + BN) * 128, pl = p.a_bytes + p.b_bytes;
    const size_t fixed = (size_t)BN * tc::kTabStride * 4 + (2 * MAXSP + 3 * MAXS + 4) * 8 + 1024;
    const size_t budget = (dual ? 112 * 1024 : 227 * 1024) - fixed;
    // operand ring S (3 stages), plane ring SP as deep
    // as the rest of shared memory allows (it hides the TMA latency); APNN_FP4_S overrides S
    int S = dual ? 2 : fp4_op_stages();
    if (S * op + 2 * pl > budget) S = (int)((budget - 2 * pl) / op);
    if (S < 2) return cudaErrorInvalidConfiguration;
    int SP = (int)((budget - S * op) / pl);
    if (SP > MAXSP) SP = MAXSP;
    if (SP < 2) return cudaErrorInvalidConfiguration;
    p.stages = S;
    p.pstages = SP;
    const size_t per_total = S * op + SP * pl;
    uint32_t cols = BN + 2 * kSfCols, pow2 = 32;
    while (pow2 < cols) pow2 <<= 1;
    p.tmem_cols = pow2;
    const size_t smem = per_total + fixed - 1024 + 64;
    CUtensorMap ta, tb;
    if (!make_map(&ta, A, g.M, g.a_bits, Kw, BM)) return cudaErrorInvalidValue;
    if (prep ? !make_map_prep(&tb, reinterpret_cast<const uint8_t*>(W), g.N, Kw, BN)
             : !make_map(&tb, reinterpret_cast<const uint32_t*>(W), g.N, g.w_bits, Kw, BN))
        return cudaErrorInvalidValue;
    dim3 grid((g.M + BM - 1) / BM, (ncols + BN - 1) / BN);
    cudaError_t err;
    if (prep) err = BN == 256 ? launch_enc<256, true>(g.enc, ta, tb, p, grid, smem, s)
                    : BN == 192 ? launch_enc<192, true>(g.enc, ta, tb, p, grid, smem, s)
                                : launch_enc<128, true>(g.enc, ta, tb, p, grid, smem, s);
    else err = BN == 256 ? launch_enc<256, false>(g.enc, ta, tb, p, grid, smem, s)
                         : launch_enc<128, false>(g.enc, ta, tb, p, grid, smem, s);
    count_launch();
    return err;
}

cudaError_t launch_tc_fp4(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                          cudaStream_t s) {
    return launch_fp4_impl(A, W, false, g, e, Y, s);
}

cudaError_t launch_tc_fp4_prepared(const uint32_t* A, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                   cudaStream_t s) {
    return launch_fp4_impl(A, Wp, true, g, e, Y, s);
}

cudaError_t launch_prepare_weights(const uint32_t* W, int N, int K, int w_bits, int enc, uint8_t* out, int sms,
                                   cudaStream_t s) {
    using namespace fp4;
    const int Kw = (K + 127) / 128 * 4;
    if ((long long)N * Kw == 0) return cudaSuccess;
    const int Kq = Kw / 4;
    // 256-thread CTAs: x over a row's 16-byte plane words, y over rows; ~8 CTAs per SM
    dim3 threads(Kq >= 256 ? 256 : (Kq + 31) / 32 * 32, 1);
    threads.y = 256 / threads.x;
    dim3 blocks((Kq + threads.x - 1) / threads.x, 1);
    long long ry = ((long long)sms * 8 + blocks.x - 1) / blocks.x;
    long long need = ((long long)N + threads.y - 1) / threads.y;
    blocks.y = (unsigned)(ry < need ? ry : need);
    if (blocks.y > 65535) blocks.y = 65535;
    const bool pm1 = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_PM1_A_01;
    if (pm1) prepare_kernel<1, true><<<blocks, threads, 0, s>>>(W, N, K, Kw, out);
    else if (w_bits == 1) prepare_kernel<1, false><<<blocks, threads, 0, s>>>(W, N, K, Kw, out);
    else prepare_kernel<2, false><<<blocks, threads, 0, s>>>(W, N, K, Kw, out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace apnn
