// gemm_tc.cu -- tcgen05 kind::i8 variant of the AP-bit contraction (APNN_VARIANT_TC_I8).
//
// How the paper's method maps to sm_100a:
// B200 has no 1-bit tensor-core MMA (kind::b1 does not exist; the legacy b1
// mma.sync is emulated on the int8 pipe).  The paper's bit combination
//     Y = sum_s sum_t 2^(s+t) W^(s) X^(t)
// is bilinear, so it equals (sum_t 2^t X^(t)) . (sum_s 2^s W^(s))^T: the
// combination can be applied to the OPERANDS (O((a+w)(M+N)K) shift-ors on the
// CUDA cores) instead of the p.q partial products (O(pq MN) adds), after which
// a single int8 tensor-core contraction per tile yields Y exactly.  +-1 planes
// decode to s8 -1/+1 (Cases II/III: the J terms disappear
// once the value is materialised); 0/1 codes are u8.
//
// Per CTA: a 128 x BN output tile, K in blocks of 128 (the paper's b_k = 128,
// PAPER.md:1742), S-stage pipeline:
//   warp 0      TMA producer: one 3-D box per operand per k-block brings ALL
//               planes of the tile ("virtual batching", PAPER.md:1528-1533:
//               the plane index is a box dimension) into shared memory.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (4 MMAs of
//               128 x BN x 32 per k-block), int32 accumulator in TMEM
//               ("fragment caching", now TMEM).
//   warps 2-9   recombination: planes -> int8.  A goes straight into TMEM with
//               tcgen05.st (the MMA's A operand is TMEM-resident), B goes into
//               the UMMA K-major no-swizzle layout in shared memory.  Then the
//               same warps run the epilogue: tcgen05.ld -> int32 store, or the
//               fused element-wise routine -> requantise -> bit-decompose ->
//               pack along N in registers.
// K ordering inside a 32-element group is permuted identically for A and B
// (word j of a group holds elements j, j+8, j+16, j+24) so that one shift +
// one masked OR per plane builds four int8 lanes.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace apnn {

namespace tc {

constexpr int BM = 128;
constexpr int NUM_RECOMB_WARPS = 8;
constexpr int NT = 32 * (2 + NUM_RECOMB_WARPS);
constexpr int MAX_STAGES = 6;

struct Params {
    Geom g;
    Epi e;
    void* Y;
    int stages;
    int nkb;            // k-blocks
    uint32_t a_bytes;   // planes bytes of A per stage
    uint32_t b_bytes;   // planes bytes of B per stage
    uint32_t tmem_cols;
};

// decode one 32-element group of 0/1 planes into 8 words of u8 lanes:
// word j, byte i <- element j + 8 i  (one shift + one masked OR per plane)
template <int NB>
__device__ __forceinline__ void decode_01(const uint32_t (&pw)[8], uint32_t (&out)[8]) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
        uint32_t o = 0;
#pragma unroll
        for (int t = 0; t < NB; t++) {
            const uint32_t mask = 0x01010101u << t;
            const uint32_t sh = (j >= t) ? (pw[t] >> (j - t)) : (pw[t] << (t - j));
            o |= sh & mask;
        }
        out[j] = o;
    }
}
__device__ __forceinline__ void decode_01_any(const uint32_t (&pw)[8], int nb, uint32_t (&out)[8]) {
    switch (nb) {  // warp-uniform
    case 1: decode_01<1>(pw, out); break;
    case 2: decode_01<2>(pw, out); break;
    case 3: decode_01<3>(pw, out); break;
    case 4: decode_01<4>(pw, out); break;
    case 5: decode_01<5>(pw, out); break;
    case 6: decode_01<6>(pw, out); break;
    case 7: decode_01<7>(pw, out); break;
    default: decode_01<8>(pw, out); break;
    }
}

// +-1 plane -> s8 lanes: bit 1 -> 0x01, bit 0 -> 0xFF; vm = valid elements
__device__ __forceinline__ void decode_pm1(uint32_t pw, uint32_t vm, uint32_t (&out)[8]) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint32_t s = (pw >> j) & 0x01010101u;
        uint32_t o = s * 0xFFFFFF02u + 0xFFFFFFFFu;  // 0xFF - 0xFE*s per byte, no borrows
        const uint32_t v = (vm >> j) & 0x01010101u;
        out[j] = o & (v * 0xFFu);
    }
}

template <int BN, bool A_PM1, bool W_PM1>
__global__ void __launch_bounds__(NT, 1)
    tc_i8_gemm_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                      const Params p) {
    using namespace sm100;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    // layout: [B operand stages][A planes stages][B planes stages][barriers]
    uint8_t* sBop = smem;                                    // S x BN x 128 B, 1024-aligned
    uint8_t* sApl = sBop + (size_t)S * BN * 128;             // S x a_bytes
    uint8_t* sBpl = sApl + (size_t)S * p.a_bytes;            // S x b_bytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(sBpl + (size_t)S * p.b_bytes);
    uint64_t* plane_full = bars;
    uint64_t* plane_empty = bars + MAX_STAGES;
    uint64_t* op_full = bars + 2 * MAX_STAGES;
    uint64_t* op_empty = bars + 3 * MAX_STAGES;
    uint64_t* accum_full = bars + 4 * MAX_STAGES;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * MAX_STAGES + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const Geom& g = p.g;
    const int nkb = p.nkb;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmapA);
        tma_prefetch(&tmapB);
        for (int s = 0; s < S; s++) {
            mbar_init(&plane_full[s], 1);
            mbar_init(&plane_empty[s], NUM_RECOMB_WARPS);
            mbar_init(&op_full[s], NUM_RECOMB_WARPS);
            mbar_init(&op_empty[s], 1);
        }
        mbar_init(accum_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_dyn(tmem_holder, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const uint32_t A_COL = BN;  // A stages live after the accumulator columns

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&plane_empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&plane_full[s], p.a_bytes + p.b_bytes);
                tma_load_3d(sApl + (size_t)s * p.a_bytes, &tmapA, &plane_full[s], kb * 4, m0, 0);
                tma_load_3d(sBpl + (size_t)s * p.b_bytes, &tmapB, &plane_full[s], kb * 4, n0, 0);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(BM, BN, A_PM1, W_PM1);
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&op_full[s], ph);
                tc_fence_after();
                const uint32_t bbase = smem_u32(sBop + (size_t)s * BN * 128);
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    const uint64_t bdesc = umma_desc_noswizzle(bbase + kk * 256, 128, 1024);
                    mma_i8_ts(tmem, tmem + A_COL + s * 32 + kk * 8, bdesc, idesc, (kb | kk) != 0);
                }
                mma_commit(&op_empty[s]);
            }
            mma_commit(accum_full);
        }
    } else {
        // ------------------------------------------------ recombination warps
        const int q = warp & 3;             // TMEM lane quarter this warp may access
        const int grp = (warp - 2) >> 2;    // 0: warps 2-5, 1: warps 6-9
        const int t = q * 32 + lane;        // row slot 0..127
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        const int ab = g.a_bits, wb = g.w_bits;

        for (int kb = 0; kb < nkb; kb++) {
            const int s = kb % S;
            const uint32_t ph = (kb / S) & 1;
            const bool doA = ((kb & 1) == grp);
            mbar_wait(&plane_full[s], ph);
            // planes of this thread's rows (smem layout [plane][row][16 B])
            uint4 pa[8];
            uint4 pb[2][8];
            if (doA) {
                const uint4* src = reinterpret_cast<const uint4*>(sApl + (size_t)s * p.a_bytes);
#pragma unroll
                for (int pl = 0; pl < 8; pl++)
                    if (pl < ab) pa[pl] = src[pl * BM + t];
            } else {
                const uint4* src = reinterpret_cast<const uint4*>(sBpl + (size_t)s * p.b_bytes);
#pragma unroll
                for (int r = 0; r < 2; r++) {
                    const int row = t + r * 128;
                    if (row < BN) {
#pragma unroll
                        for (int pl = 0; pl < 8; pl++)
                            if (pl < wb) pb[r][pl] = src[pl * BN + row];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&plane_empty[s]);

            mbar_wait(&op_empty[s], ph ^ 1);
            // valid-element mask for +-1 x +-1 (Case II): padded K must decode to 0
            int kvalid = 128;
            if (A_PM1 && W_PM1) {
                const int rem = g.K - kb * 128;
                kvalid = rem < 128 ? rem : 128;
            }
            if (doA) {
#pragma unroll
                for (int gi = 0; gi < 4; gi++) {
                    uint32_t pw[8];
#pragma unroll
                    for (int pl = 0; pl < 8; pl++) {
                        const uint4 v = pa[pl < ab ? pl : 0];
                        pw[pl] = gi == 0 ? v.x : gi == 1 ? v.y : gi == 2 ? v.z : v.w;
                    }
                    uint32_t o[8];
                    if (A_PM1) {
                        const int nv = kvalid - gi * 32;
                        const uint32_t vm = nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
                        decode_pm1(pw[0], vm, o);
                    } else {
                        decode_01_any(pw, ab, o);
                    }
                    tmem_st8(tmem_lane + A_COL + s * 32 + gi * 8, o);
                }
                tmem_wait_st();
            } else {
                uint8_t* dst = sBop + (size_t)s * BN * 128;
#pragma unroll
                for (int r = 0; r < 2; r++) {
                    const int row = t + r * 128;
                    if (row >= BN) continue;
                    uint8_t* rbase = dst + (row >> 3) * 1024 + (row & 7) * 16;
#pragma unroll
                    for (int gi = 0; gi < 4; gi++) {
                        uint32_t pw[8];
#pragma unroll
                        for (int pl = 0; pl < 8; pl++) {
                            const uint4 v = pb[r][pl < wb ? pl : 0];
                            pw[pl] = gi == 0 ? v.x : gi == 1 ? v.y : gi == 2 ? v.z : v.w;
                        }
                        uint32_t o[8];
                        if (W_PM1) decode_pm1(pw[0], 0xFFFFFFFFu, o);
                        else decode_01_any(pw, wb, o);
                        *reinterpret_cast<uint4*>(rbase + (2 * gi) * 128) = make_uint4(o[0], o[1], o[2], o[3]);
                        *reinterpret_cast<uint4*>(rbase + (2 * gi + 1) * 128) = make_uint4(o[4], o[5], o[6], o[7]);
                    }
                }
                fence_proxy_async_smem();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&op_full[s]);
        }

        // ------------------------------------------------ epilogue
        mbar_wait(accum_full, 0);
        tc_fence_after();
        const int m = m0 + t;
        const Epi& e = p.e;
        const int ncol_half = BN / 2;
        for (int c = grp * ncol_half; c < (grp + 1) * ncol_half; c += 32) {
            uint32_t acc[32];
            tmem_ld32(tmem_lane + c, acc);
            tmem_wait_ld();
            const int nb = n0 + c;
            if (m >= g.M) continue;
            if (e.out_bits == 0) {
                int32_t* Y = reinterpret_cast<int32_t*>(p.Y) + (long long)m * g.N;
                if (nb + 32 <= g.N && (g.N & 3) == 0) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        *reinterpret_cast<int4*>(Y + nb + i) =
                            make_int4((int)acc[i], (int)acc[i + 1], (int)acc[i + 2], (int)acc[i + 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; i++)
                        if (nb + i < g.N) Y[nb + i] = (int)acc[i];
                }
            } else {
                const int Nw = (g.N + 127) / 128 * 4;
                const int word = nb / 32;
                if (word >= Nw) continue;
                uint32_t qb[8];
#pragma unroll
                for (int i = 0; i < 8; i++) qb[i] = 0;
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    const int n = nb + i;
                    uint32_t qv = 0;
                    if (n < g.N) qv = requant(e, (int32_t)acc[i], epi_alpha(e, n), epi_beta(e, n));
                    qb[i >> 2] |= qv << (8 * (i & 3));
                }
                uint32_t* o = reinterpret_cast<uint32_t*>(p.Y) + (long long)m * e.out_bits * Nw + word;
                for (int tb = 0; tb < e.out_bits; tb++) {
                    uint32_t wv = 0;
#pragma unroll
                    for (int qq = 0; qq < 8; qq++) wv |= byte_bits_to_nibble(qb[qq], tb) << (4 * qq);
                    o[(long long)tb * Nw] = wv;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, p.tmem_cols);
    }
}

// ------------------------------------------------------------------ host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
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

// Packed operand [rows][bits][Cw] viewed as a 3-D uint32 tensor {Cw, rows, bits}
// (dims listed innermost first); box {4 words = 128 elements, box_rows, bits}
// lands in shared memory as [plane][row][16 B].
static bool make_plane_map(CUtensorMap* m, const uint32_t* base, int rows, int bits, int Cw, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)Cw, (cuuint64_t)rows, (cuuint64_t)bits};
    cuuint64_t strides[2] = {(cuuint64_t)bits * Cw * 4, (cuuint64_t)Cw * 4};
    cuuint32_t box[3] = {4, (cuuint32_t)box_rows, (cuuint32_t)bits};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace tc

bool tc_i8_supports(const Geom& g) {
    // GEMM only for now (conv runs on the popc variant); K = 0 has no MMA to issue
    return !g.conv && g.K > 0 && g.M > 0 && g.N > 0;
}

template <int BN, bool AP, bool WP>
static cudaError_t launch_tc_t(const CUtensorMap& ta, const CUtensorMap& tb, const tc::Params& p, dim3 grid,
                               size_t smem, cudaStream_t s) {
    auto kfn = tc::tc_i8_gemm_kernel<BN, AP, WP>;
    static bool attr_set = false;  // per-instantiation; benign race (same value)
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    kfn<<<grid, tc::NT, smem, s>>>(ta, tb, p);
    return cudaGetLastError();
}

template <int BN>
static cudaError_t launch_tc_bn(const CUtensorMap& ta, const CUtensorMap& tb, const tc::Params& p, dim3 grid,
                                size_t smem, cudaStream_t s) {
    switch (p.g.enc) {
    case APNN_ENC_01_01: return launch_tc_t<BN, false, false>(ta, tb, p, grid, smem, s);
    case APNN_ENC_PM1_PM1: return launch_tc_t<BN, true, true>(ta, tb, p, grid, smem, s);
    case APNN_ENC_W_PM1_A_01: return launch_tc_t<BN, false, true>(ta, tb, p, grid, smem, s);
    default: return launch_tc_t<BN, true, false>(ta, tb, p, grid, smem, s);
    }
}

cudaError_t launch_tc_i8(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y, int sms,
                         cudaStream_t s) {
    (void)sms;
    const int BN = g.N > 128 ? 256 : (g.N > 64 ? 128 : 64);
    tc::Params p;
    p.g = g;
    p.e = e;
    p.Y = Y;
    p.nkb = g.nchunks;
    p.a_bytes = 16u * tc::BM * g.a_bits;
    p.b_bytes = 16u * BN * g.w_bits;
    const size_t per_stage = (size_t)BN * 128 + p.a_bytes + p.b_bytes;
    const size_t budget = 227 * 1024 - 1024 - 256;
    int S = (int)(budget / per_stage);
    if (S > tc::MAX_STAGES) S = tc::MAX_STAGES;
    if (S < 2) return cudaErrorInvalidConfiguration;
    p.stages = S;
    uint32_t cols = BN + 32 * S;
    uint32_t pow2 = 32;
    while (pow2 < cols) pow2 <<= 1;
    p.tmem_cols = pow2;
    const size_t smem = (size_t)S * per_stage + (4 * tc::MAX_STAGES + 2) * 8 + 64;

    CUtensorMap ta, tb;
    if (!tc::make_plane_map(&ta, A, g.M, g.a_bits, g.Cw, tc::BM)) return cudaErrorInvalidValue;
    if (!tc::make_plane_map(&tb, W, g.N, g.w_bits, g.Cw, BN)) return cudaErrorInvalidValue;

    const int ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;
    dim3 grid((g.M + tc::BM - 1) / tc::BM, (ncols + BN - 1) / BN);
    cudaError_t err;
    if (BN == 256) err = launch_tc_bn<256>(ta, tb, p, grid, smem, s);
    else if (BN == 128) err = launch_tc_bn<128>(ta, tb, p, grid, smem, s);
    else err = launch_tc_bn<64>(ta, tb, p, grid, smem, s);
    count_launch();
    return err;
}

}  // namespace apnn
