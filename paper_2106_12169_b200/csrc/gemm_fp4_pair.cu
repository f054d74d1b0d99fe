// gemm_fp4_pair.cu -- persistent CTA-pair version of the exact-FP4 contraction (row f3;
// the bench GEMM: apnn_gemm_prepared).
//
// Same arithmetic as gemm_fp4.cu: the bit combination of PAPER.md:1426-1429 applied to the
// operands, <= 2-bit codes as e2m1 values, `tcgen05.mma kind::mxf4.block_scale` with unit
// E8M0 scales, fp32 accumulation exact below 2^24 (host bound, adversarial tests in
// tests/test_fp4_exact.py).  What changes is the mapping onto the machine:
//
//   * CTA pairs (cta_group::2): a 256 x BNP output tile per pair, A rows split across the
//     two CTAs (128 each), the prepared W rows split too (BNP/2 each), so every SM stages
//     half the W bytes of a one-CTA 128 x BNP tile for the same MMA work;
//   * persistent: one pair per two SMs loops over tiles; with BNP = 224 the TMEM holds two
//     224-column accumulators (+ the scale-factor columns), so the epilogue of tile i
//     overlaps the MMAs of tile i+1;
//   * A at half scale: code v is stored as the e2m1 value v/2 (0, .5, 1, 1.5), whose nibble
//     is the code itself -- one shift and mask per plane and word, no table (+-1 -> +-0.5:
//     0x1 / 0x9).  The accumulator then holds Y/2 (half-integers, exact while |Y| < 2^24)
//     and the epilogue doubles it exactly.
//
// Warp roles per CTA (19 warps):
//   warps 0-7    A recombination in two teams of 4 on alternating stages (two stages in
//                flight per SM sub-partition): packed planes (TMA ring) -> e2m1 nibbles in
//                the K-major SWIZZLE_128B A operand stage; a lane pair covers two rows x the
//                stage's two k-blocks of 128
//   warps 8-15   epilogue (two warps per TMEM lane quarter, each half of the columns):
//                tcgen05.ld -> x2 -> int32, or the fused requantise + pack of tc_common.cuh
//   warp 16      TMA producer of the A planes (4 lanes side by side; runs up to SP stages ahead)
//   warp 17      TMA producer of this CTA's prepared-W half, straight into the operand ring
//   warp 18      TMEM allocator; in CTA 0 the single-thread MMA issuer
#include <cuda.h>

#include <cstdio>
#include <cstring>

#include "tc_common.cuh"

namespace apnn {
namespace fp4 {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool make_map(CUtensorMap* m, const uint32_t* base, int rows, int bits, int Kw, int box_rows);
bool make_map_prep(CUtensorMap* m, const uint8_t* base, int N, int Kw, int box_rows);
bool make_map_rows(CUtensorMap* m, const uint8_t* base, int rows, int row_bytes, int box_rows);

namespace pair {

using namespace sm100;

// Experiment builds only (build.py --variant NAME -DAPNN_EXP_PAIR=n; wrong results by design):
//   1 decode warps skip the plane loads / decode / operand stores (barrier protocol kept)
//   2 the MMA issuer commits without issuing MMAs
//   3 the W producer arrives without loading (no W traffic)
//   4 the A-plane producer arrives without loading (no A traffic); 5 = 3 + 4
#ifndef APNN_EXP_PAIR
#define APNN_EXP_PAIR 0
#endif
// APNN_EXP_PAIR_TRACE=1 (experiment builds): clock64 stamps of CTA 0's pipeline events,
// read back with apnn_exp_pair_trace()
#ifndef APNN_EXP_PAIR_TRACE
#define APNN_EXP_PAIR_TRACE 0
#endif
enum { TR_PA = 0, TR_PB, TR_PLANE, TR_OPEMPTY, TR_ARRIVE, TR_MMAWAIT, TR_MMADONE, TR_EPI0, TR_EPIREL, TR_EPIEND,
       TR_WARR = 10, TR_NEV = TR_WARR + 32 };  // TR_WARR + 8 * cta + 4 * (what) + team-warp: per-warp stamps
constexpr int kTrN = 1024;
#if APNN_EXP_PAIR_TRACE
__device__ unsigned long long g_trace[TR_NEV * kTrN];
#endif
// CTA 0 stamps clock64; CTA 1's per-warp stamps use %globaltimer-free clock64 too (SM clocks
// are not synchronised, so only intervals within one CTA are compared)
__device__ __forceinline__ void tr(int ev, int i) {
#if APNN_EXP_PAIR_TRACE
    if (blockIdx.x == 0 && i < kTrN) g_trace[ev * kTrN + i] = clock64();
#endif
}
__device__ __forceinline__ void trg(int ev, int i) {  // both CTAs of pair 0, globaltimer (ns)
#if APNN_EXP_PAIR_TRACE
    if (blockIdx.x < 2 && i < kTrN) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[ev * kTrN + i] = t;
    }
#endif
}

constexpr int DEC_WARPS = 8;
constexpr int EPI_WARPS = 8;
constexpr int EPI0 = DEC_WARPS;
constexpr int TMA_WARP = EPI0 + EPI_WARPS;  // A planes
constexpr int TMB_WARP = TMA_WARP + 1;      // prepared W
constexpr int MMA_WARP = TMB_WARP + 1;
constexpr int TEAM_WARPS = DEC_WARPS / 2;
constexpr int THREADS = (MMA_WARP + 1) * 32;
constexpr int MAXS = 8;    // A operand stages (decoded e2m1, 16 KB each)
constexpr int MAXSB = 10;  // W operand stages (prepared e2m1 half, TMA; the deep ring: L2 latency)
constexpr int MAXSP = 12;  // A plane stages
constexpr int kProdLanes = 4;
constexpr uint32_t AOP = 128 * 128;  // A operand stage: 128 rows x 128 bytes (256 e2m1)

struct Params {
    Geom g;
    Epi e;
    void* Y;
    int S, SB, SP;    // A operand / W operand / A plane ring depths
    int nst;          // stages (256 K elements) per tile
    uint32_t a_bytes; // A plane bytes per stage (128 rows x a_bits x 32 B)
    int tiles_m, tiles_n, num_tiles;
    int tab_mode;
    int stg_warp;     // epilogue staging bytes per warp
    int ncols;        // columns the tiles cover (int32: N; packed: Nw * 32)
    uint32_t idesc;   // pp kernel, kind::i8: the instruction descriptor (operand signedness)
};

__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma2_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                          uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// 32 elements of one group (plane words pw) -> 4 words of e2m1 nibbles at HALF scale;
// word j holds elements j, j+4, ..., j+28 (the element order of gemm_fp4.cu and of the
// prepared W, so the dot product is unchanged)
template <int NB, bool PM1>
__device__ __forceinline__ void decode_group_half(const uint32_t (&pw)[2], uint32_t (&o)[4]) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
        uint32_t w;
        if (PM1) {  // +1 -> +0.5 (0x1), -1 -> -0.5 (0x9)
            w = 0x11111111u | (((~pw[0] >> j) & 0x11111111u) << 3);
        } else if (NB == 1) {  // 0 -> 0, 1 -> 0.5 (0x1)
            w = (pw[0] >> j) & 0x11111111u;
        } else {  // v -> v/2: nibble = (bit1 << 1) | bit0
            const uint32_t hi = j ? (pw[1] >> (j - 1)) : (pw[1] << 1);
            w = ((pw[0] >> j) & 0x11111111u) | (hi & 0x22222222u);
        }
        o[j] = w;
    }
}

// one lane: rows r and r + 16 of the stage, k-block kb2 (its plane chunks at byte offset
// src_off and src_off + 512 of the plane stage [plane][128 rows][2 x 16 B])
template <int NB, bool PM1>
__device__ __forceinline__ void decode_job2(const uint8_t* planes, uint32_t src_off, uint32_t (&o)[2][4][4],
                                            volatile uint32_t* dep_slot) {
    uint4 v[2][NB];
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
        for (int pl = 0; pl < NB; pl++)
            v[j][pl] = *reinterpret_cast<const uint4*>(planes + src_off + j * 512 + pl * 4096);
    // the plane-stage release after this call must not overtake these loads (tc_common.cuh recomb_step)
    uint32_t dep = 0;
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
        for (int pl = 0; pl < NB; pl++) dep ^= v[j][pl].x;
    *dep_slot = dep;
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
        for (int gi = 0; gi < 4; gi++) {
            uint32_t pw[2] = {0u, 0u};
#pragma unroll
            for (int pl = 0; pl < NB; pl++) pw[pl] = tc::sel4(v[j][pl], gi);
            decode_group_half<NB, PM1>(pw, o[j][gi]);
        }
}

// long waits (the epilogue idles most of a tile): back off instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) __nanosleep(100);
}

// staged packed words [32 rows][ob][nwb] -> out[(row * ob + t) * Nw + w0 + w] (clipped)
__device__ __forceinline__ void writeback_words(const uint32_t* stg, int lane, uint32_t* out, int row0, int row_end,
                                                int w0, int Nw, int ob, int nwb) {
    const int per_row = ob * nwb, total = 32 * per_row;
    for (int i = lane; i < total; i += 32) {
        const int r = i / per_row, rem = i - r * per_row;
        const int t = rem / nwb, w = rem - t * nwb;
        if (row0 + r < row_end && w0 + w < Nw) out[((long long)(row0 + r) * ob + t) * Nw + w0 + w] = stg[i];
    }
}

template <int BNP, bool A_PM1, bool W_PM1, bool I32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    fp4_pair_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                    const Params p) {
    constexpr int BROWS = BNP / 2;                   // prepared W rows per CTA
    constexpr uint32_t BOP = BROWS * 128;            // W operand stage bytes
    constexpr int NACC = (2 * BNP + 64 <= 512) ? 2 : 1;
    constexpr uint32_t SFA = (uint32_t)(NACC * BNP + 31) / 32 * 32, SFB = SFA + 32;
    constexpr int NCK = BNP / 32;                    // 32-column chunks per tile
    constexpr int NCK0 = (NCK + 1) / 2;              // chunks of the first epilogue half
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.S, SB = p.SB, SP = p.SP;
    uint8_t* sAop = smem;                                        // S x 16 KB
    uint8_t* sBop = sAop + (size_t)S * AOP;                      // SB x BOP
    uint8_t* sApl = sBop + (size_t)SB * BOP;                     // SP x a_bytes
    uint8_t* sStg = sApl + (size_t)SP * p.a_bytes;               // EPI_WARPS x stg_warp
    int32_t* sTab = reinterpret_cast<int32_t*>(sStg + (size_t)EPI_WARPS * p.stg_warp);  // BNP x kTabStride
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + (I32 ? 0 : BNP * tc::kTabStride));  // int32: no table
    uint64_t* plane_full = bars;                  // [MAXSP]
    uint64_t* plane_empty = bars + MAXSP;         // [MAXSP]
    uint64_t* op_full = bars + 2 * MAXSP;         // [MAXS] (CTA 0: both CTAs' A writers, W landed)
    uint64_t* op_empty = op_full + MAXS;          // [MAXS] A stage consumed (multicast MMA commit)
    uint64_t* b_full = op_empty + MAXS;           // [MAXSB] this CTA's W half landed
    uint64_t* b_empty = b_full + MAXSB;           // [MAXSB] W stage consumed (multicast MMA commit)
    uint64_t* accum_full = b_empty + MAXSB;       // [2]
    uint64_t* accum_empty = accum_full + 2;       // [2] (CTA 0: both CTAs' epilogue warps)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accum_empty + 2);
    volatile uint32_t* dep_slots = tmem_holder + 1;  // [DEC_WARPS * 32]

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const Geom& g = p.g;
    const int nst = p.nst;

    if (warp == TMA_WARP && lane == 0) {
        tma_prefetch(&tmapA);
        tma_prefetch(&tmapB);
        for (int s = 0; s < SP; s++) {
            mbar_init(&plane_full[s], 1);
            mbar_init(&plane_empty[s], TEAM_WARPS);
        }
        for (int s = 0; s < S; s++) {
            mbar_init(&op_full[s], 2 * TEAM_WARPS);
            mbar_init(&op_empty[s], 1);
        }
        for (int s = 0; s < SB; s++) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&accum_full[i], 1);
            mbar_init(&accum_empty[i], 2 * EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == MMA_WARP) tmem_alloc2(tmem_holder, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    if (warp >= EPI0 && warp < EPI0 + 4) {  // every scale-factor byte = E8M0 127 (2^0), all lanes, both CTAs
        const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t ones[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
#pragma unroll
        for (uint32_t c = 0; c < 64; c += 8) tmem_st8(lb + SFA + c, ones);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();

    if (warp == TMA_WARP || warp == TMB_WARP) {
        // ------------------------------------------------------------ TMA producers
        // lanes 0..3 issue consecutive stages side by side (hides the per-stage barrier
        // round trip of one issuing thread, gemm_tc.cu); A planes and W halves run
        // independently, so the plane ring fills SP stages ahead of the operand ring
        const bool is_a = warp == TMA_WARP;
        const int my_tiles = p.num_tiles > cid ? (p.num_tiles - cid + ncl - 1) / ncl : 0;
        const int total = my_tiles * nst;
        for (int base = 0; base < total; base += kProdLanes) {
            const int it = base + lane;
            if (lane < kProdLanes && it < total) {
                const int ti = it / nst, st = it - ti * nst;
                const int tile = cid + ti * ncl;
                const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
                if (is_a) {
                    const int ps = it % SP;
                    const uint32_t pph = (uint32_t)(it / SP) & 1u;
                    mbar_wait(&plane_empty[ps], pph ^ 1);
                    tr(TR_PA, it);
#if APNN_EXP_PAIR == 4 || APNN_EXP_PAIR == 5
                    mbar_arrive(&plane_full[ps]);
#else
                    mbar_arrive_expect_tx(&plane_full[ps], p.a_bytes);
                    tma_load_4d(sApl + (size_t)ps * p.a_bytes, &tmapA, &plane_full[ps], st * 8,
                                (tm * 2 + (int)rank) * 128, 0, 0);
#endif
                } else {
                    const int os = it % SB;
                    const uint32_t oph = (uint32_t)(it / SB) & 1u;
                    mbar_wait(&b_empty[os], oph ^ 1);
                    tr(TR_PB, it);
#if APNN_EXP_PAIR == 3 || APNN_EXP_PAIR == 5
                    mbar_arrive(&b_full[os]);
#else
                    mbar_arrive_expect_tx(&b_full[os], BOP);
                    tma_load_2d(sBop + (size_t)os * BOP, &tmapB, &b_full[os], st * 128, tn * BNP + (int)rank * BROWS);
#endif
                }
            }
            __syncwarp();
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer (CTA 0)
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = idesc_mxf4(256, BNP);
            const uint32_t a0 = smem_u32(sAop), b0 = smem_u32(sBop);
            int s = 0, sb = 0, tc = 0, itm = 0;
            uint32_t ph = 0;
            for (int tile = cid; tile < p.num_tiles; tile += ncl, tc++) {
                const int buf = NACC == 2 ? (tc & 1) : 0;
                mbar_wait_cluster(&accum_empty[buf], ((tc / NACC) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * BNP);
                for (int st = 0; st < nst; st++) {
                    mbar_wait_cluster(&op_full[s], ph);
                    tr(TR_MMAWAIT, itm);
                    trg(TR_WARR + 12, itm);
                    tc_fence_after();
                    const uint32_t ab = a0 + (uint32_t)s * AOP, bb = b0 + (uint32_t)sb * BOP;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)  // K = 64 e2m1 elements = 32 bytes per MMA
                        if (APNN_EXP_PAIR != 2) mma2_mxf4(d, tc::b_desc(ab, kk), tc::b_desc(bb, kk), idesc, tmem + SFA, tmem + SFB,
                                  (st | kk) != 0);
                    mma2_commit_mc(&op_empty[s], 0x3);
                    mma2_commit_mc(&b_empty[sb], 0x3);
                    tr(TR_MMADONE, itm++);
                    if (++s == S) { s = 0; ph ^= 1; }
                    if (++sb == SB) sb = 0;
                }
                mma2_commit_mc(&accum_full[buf], 0x3);
            }
        }
    } else if (warp < DEC_WARPS) {
        // ------------------------------------------------------------ A recombination
        const int team = warp / TEAM_WARPS;
        const int r0 = (warp % TEAM_WARPS) * 32 + (lane >> 1), kb2 = lane & 1;
        // planes: row r, k-block kb2 of plane pl at byte (pl * 128 + r) * 32 + kb2 * 16;
        // operand: chunk c of row r at tc::b_chunk_offset(r, c); row r + 16 is 2048 bytes on
        const uint32_t src_off = (uint32_t)(r0 * 32 + kb2 * 16);
        uint32_t dst_off[4];
#pragma unroll
        for (int gi = 0; gi < 4; gi++) dst_off[gi] = tc::b_chunk_offset(r0, kb2 * 4 + gi);
        const uint32_t op_full0 = mapa(smem_u32(op_full), 0);
        const int a_bits = g.a_bits;
        int s = 0, ps = 0, sb = 0, it = 0;
        uint32_t ph = 0, pph = 0, bph = 0;
        for (int tile = cid; tile < p.num_tiles; tile += ncl) {
            for (int st = 0; st < nst; st++, it++, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0),
                     ps = (ps + 1 == SP) ? 0 : ps + 1, pph ^= (ps == 0), sb = (sb + 1 == SB) ? 0 : sb + 1,
                     bph ^= (sb == 0)) {
                if ((it & 1) != team) continue;
                mbar_wait(&plane_full[ps], pph);
                if ((warp & 3) == 0 && lane == 0) tr(TR_PLANE, it);
                if (lane == 0) trg(TR_WARR + 16 * blockIdx.x + 8 + (warp & 3), it);
                uint32_t o[2][4][4];
                const uint8_t* pl = sApl + (size_t)ps * p.a_bytes;
                if (APNN_EXP_PAIR == 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&plane_empty[ps]);
                    mbar_wait(&op_empty[s], ph ^ 1);
                    mbar_wait(&b_full[sb], bph);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(op_full0 + (uint32_t)s * 8u);
                    continue;
                }
                if (A_PM1) decode_job2<1, true>(pl, src_off, o, dep_slots + threadIdx.x);
                else if (a_bits == 1) decode_job2<1, false>(pl, src_off, o, dep_slots + threadIdx.x);
                else decode_job2<2, false>(pl, src_off, o, dep_slots + threadIdx.x);
                __syncwarp();
                if (lane == 0) mbar_arrive(&plane_empty[ps]);
                mbar_wait(&op_empty[s], ph ^ 1);
                if ((warp & 3) == 0 && lane == 0) tr(TR_OPEMPTY, it);
                if (lane == 0) trg(TR_WARR + 16 * blockIdx.x + 4 * 0 + (warp & 3) + 8 * 0, it);
                uint8_t* aop = sAop + (size_t)s * AOP;
#pragma unroll
                for (int j = 0; j < 2; j++)
#pragma unroll
                    for (int gi = 0; gi < 4; gi++)
                        *reinterpret_cast<uint4*>(aop + dst_off[gi] + j * 2048) =
                            make_uint4(o[j][gi][0], o[j][gi][1], o[j][gi][2], o[j][gi][3]);
                fence_proxy_async_smem();
                mbar_wait(&b_full[sb], bph);  // this CTA's W half of the stage has landed
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(op_full0 + (uint32_t)s * 8u);
                if ((warp & 3) == 0 && lane == 0) tr(TR_ARRIVE, it);
                if (lane == 0) trg(TR_WARR + 16 * blockIdx.x + 4 * 1 + (warp & 3), it);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;                  // TMEM lane quarter
        const int half = (warp - EPI0) >> 2;     // column half
        const int et = threadIdx.x - EPI0 * 32;  // 0..255
        const int c_begin = half ? NCK0 : 0, c_end = half ? NCK : NCK0;
        const int nwb = c_end - c_begin;
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t accum_empty0 = mapa(smem_u32(accum_empty), 0);
        const int ob = p.e.out_bits;
        const int Nw = (g.N + 127) / 128 * 4;
        uint8_t* stg = sStg + (size_t)(warp - EPI0) * p.stg_warp;
        int tc = 0;
        for (int tile = cid; tile < p.num_tiles; tile += ncl, tc++) {
            const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
            const int row0 = (tm * 2 + (int)rank) * 128 + q * 32;
            const int n0 = tn * BNP;
            if (!I32 && (p.tab_mode == tc::kTabQ3 || p.tab_mode == tc::kTabHybrid)) {
                named_bar_sync(1, EPI_WARPS * 32);  // the previous tile's table readers are done
                if (et < BNP) tc::build_threshold_row(sTab + et * tc::kTabStride, n0 + et, g.N, p.e);
                named_bar_sync(1, EPI_WARPS * 32);
            }
            const int buf = NACC == 2 ? (tc & 1) : 0;
            mbar_wait_sleep(&accum_full[buf], (uint32_t)(tc / NACC) & 1u);
            if (warp == EPI0 && lane == 0) tr(TR_EPI0, tc);
            tc_fence_after();
#pragma unroll 1
            for (int c = c_begin; c < c_end; c++) {
                uint32_t acc[32];
                tmem_ld32(tmem_lane + (uint32_t)(buf * BNP + c * 32), acc);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; i++)  // the accumulator holds Y/2 exactly (A at half scale)
                    acc[i] = (uint32_t)__float2int_rn(__uint_as_float(acc[i]) * 2.0f);
                if (I32) {
                    if (row0 < g.M) {
                        if ((g.N & 3) == 0) {
                            tc::stage_int32_chunk(acc, stg, lane);
                            __syncwarp();
                            tc::writeback_int32_block(stg, lane, reinterpret_cast<int32_t*>(p.Y), row0, g.M,
                                                      n0 + c * 32, g.N);
                            __syncwarp();
                        } else {
                            tc::epilogue_chunk(acc, row0 + lane, n0 + c * 32, c * 32, g, p.e, p.Y, nullptr,
                                               tc::kTabNone);
                        }
                    }
                } else {
                    uint32_t w[8];
                    if (p.tab_mode == tc::kTabQ3) {
                        tc::requant_chunk_words_q3(acc, sTab, c * 32, w[0], w[1]);
                    } else {
                        tc::requant_chunk(acc, n0 + c * 32, c * 32, g, p.e, sTab, p.tab_mode, w);
                    }
                    uint32_t* srow = reinterpret_cast<uint32_t*>(stg) + lane * ob * nwb + (c - c_begin);
#pragma unroll
                    for (int tb = 0; tb < 8; tb++)
                        if (tb < ob) srow[tb * nwb] = w[tb];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(accum_empty0 + 8u * (uint32_t)buf);
            if (warp == EPI0 && lane == 0) tr(TR_EPIREL, tc);
            if (!I32 && row0 < g.M) {
                __syncwarp();
                writeback_words(reinterpret_cast<const uint32_t*>(stg), lane, reinterpret_cast<uint32_t*>(p.Y), row0,
                                g.M, n0 / 32 + c_begin, Nw, ob, nwb);
            }
            if (warp == EPI0 && lane == 0) tr(TR_EPIEND, tc);
            __syncwarp();
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc2(tmem, 512);
    }
}

// ---------------------------------------------------------------------------------------------
// Both operands prepared (apnn_gemm_prepared_ab): A's e2m1 rows come from apnn_prepare_activations
// (the planes decoded ONCE per GEMM instead of once per N tile), so the main loop has no CUDA-core
// hand-off at all -- TMA lands A and W straight in the operand layout, and the MMA issuer waits on
// one barrier per stage in CTA 0 that both CTAs' TMA loads complete (.cta_group::2 TMA).
// Both operands are at full scale: the accumulator holds Y itself.
//
// Warp roles per CTA: warps 0..PP_EPI-1 epilogue (PP_EPI / 4 warps per TMEM lane quarter, each
// a slice of the columns); warp PP_EPI TMA producer (one lane); warp PP_EPI+1 TMEM allocator and,
// in CTA 0, the single-thread MMA issuer.
//
// Experiment builds only (build.py --variant NAME -DAPNN_EXP_PP=n; wrong results by design):
//   1 the epilogue releases the accumulator without reading it (no output)
//   2 the MMA issuer commits without issuing MMAs
//   3 the producer arrives without loading (no operand traffic); 4 = 1 + 3
//   5 = 4 + the issuer neither waits on the stage barriers nor fences; 6 = 4 + no fence;
//   7 = 5 + no producer and no threshold tables (the issuer and the accumulator hand-off alone)
#ifndef APNN_EXP_PP
#define APNN_EXP_PP 0
#endif
// APNN_EXP_PP_TRACE=1 (experiment builds): CTA 0's issuer stamps clock64 / %globaltimer around
// each stage (wait start, wait done, MMAs + commit issued) and epilogue warp 0 around each tile;
// read back with apnn_exp_pp_trace()
#ifndef APNN_EXP_PP_TRACE
#define APNN_EXP_PP_TRACE 0
#endif
constexpr int kPpTrN = 1024;
#if APNN_EXP_PP_TRACE
__device__ unsigned long long g_pp_trace[8 * kPpTrN];
#endif
__device__ __forceinline__ void pp_tr(int ev, int i) {
#if APNN_EXP_PP_TRACE
    if (blockIdx.x == 0 && i < kPpTrN) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_pp_trace[(2 * ev) * kPpTrN + i] = clock64();
        g_pp_trace[(2 * ev + 1) * kPpTrN + i] = t;
    }
#endif
}
// 8 epilogue warps (two per TMEM lane quarter): with the accumulator double-buffered their drain
// hides behind the next tile's MMAs, and 16 took issue slots from the lone MMA-issuing thread on
// its sub-partition (8192^3 w4a4 int8 fused 0.332 -> 0.319 ms with 8)
constexpr int PP_EPI = 8;
constexpr int PP_TMA = PP_EPI;
constexpr int PP_MMA = PP_EPI + 1;
constexpr int PP_THREADS = (PP_MMA + 1) * 32;
constexpr int PP_MAXS = 8;

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}

// I8: the same kernel on kind::i8 (int8 operand rows from apnn_prepare_weights_i8 /
// apnn_prepare_activations_i8, int32 accumulators, no scale factors): a 128-byte box is 128 K
// elements instead of 256, the descriptors and the stage walk are the same
//
// MC: clusters of two CTA pairs that work on vertically adjacent tiles (tm, tm + 1) of the same
// N tile; the W operand is loaded once per cluster and multicast to both pairs (CTA r of pair 0
// issues W half r into CTA r and CTA r + 2), halving W's L2 -> SM traffic; a stage slot is freed
// only when both pairs' MMAs are done with it (the empty barriers count both pairs' commits).
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const void* tmap, uint32_t bar_cluster, int c0, int c1,
                                                    uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster.cta_group::2 "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

template <int BNP, bool I32, bool I8, bool MC>
__global__ void __launch_bounds__(PP_THREADS, 1)
    fp4_pp_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                  const Params p) {
    constexpr int BROWS = BNP / 2;
    constexpr uint32_t BOP = BROWS * 128;
    // a stage is K = 512: two 128-byte TMA boxes of each operand, 8 MMAs per barrier hand-off (the
    // issuer pays ~590 cycles per hand-off whatever its MMA work, scripts/pp_trace.py: with 4 MMAs
    // of 448-512 cycles per stage it, not the tensor pipe, set the pace)
    constexpr uint32_t AST = 2 * AOP, BST = 2 * BOP;
    // two accumulators when they leave room for the scale-factor columns (32 + 32; kind::i8: none)
    constexpr int NACC = (2 * BNP + (I8 ? 0 : 64) <= 512) ? 2 : 1;
    constexpr uint32_t SFA = (uint32_t)(NACC * BNP + 31) / 32 * 32, SFB = SFA + 32;
    static_assert(I8 || SFB + 32 <= 512, "TMEM budget");
    constexpr int NCK = BNP / 32;
    constexpr int QW = PP_EPI / 4;  // epilogue warps per lane quarter
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.S;
    uint8_t* sAop = smem;                                   // S x AST
    uint8_t* sBop = sAop + (size_t)S * AST;                 // S x BST
    uint8_t* sStg = sBop + (size_t)S * BST;                 // PP_EPI x stg_warp
    int32_t* sTab = reinterpret_cast<int32_t*>(sStg + (size_t)PP_EPI * p.stg_warp);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + (I32 ? 0 : BNP * tc::kTabStride));
    uint64_t* full = bars;                   // [PP_MAXS] (CTA 0: both CTAs' A + W bytes)
    uint64_t* empty = bars + PP_MAXS;        // [PP_MAXS] (multicast MMA commit)
    uint64_t* accum_full = empty + PP_MAXS;  // [2]
    uint64_t* accum_empty = accum_full + 2;  // [2] (CTA 0: both CTAs' epilogue warps)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accum_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr int CL = MC ? 4 : 2;                     // CTAs per cluster
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = crank & 1u;                  // rank within the CTA pair
    const uint32_t lead = crank & ~1u;                 // the pair's leader (barriers, MMA issue)
    const int pic = MC ? (int)(crank >> 1) : 0;        // pair within the cluster
    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    const int units_m = MC ? p.tiles_m / 2 : p.tiles_m;
    const int num_units = units_m * p.tiles_n;
    const Geom& g = p.g;
    const int nst = p.nst;

    if (warp == PP_TMA && lane == 0) {
        tma_prefetch(&tmapA);
        tma_prefetch(&tmapB);
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC ? 2 : 1);  // both pairs' commits
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&accum_full[i], 1);
            mbar_init(&accum_empty[i], 2 * PP_EPI);
        }
        fence_mbar_init();
    }
    if (warp == PP_MMA) tmem_alloc2(tmem_holder, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    if (!I8 && warp < 4) {  // every scale-factor byte = E8M0 127 (2^0), all lanes, both CTAs
        const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
        const uint32_t ones[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
#pragma unroll
        for (uint32_t c = 0; c < 64; c += 8) tmem_st8(lb + SFA + c, ones);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();

    if (warp == PP_TMA) {
        // ------------------------------------------------------------ TMA producer (A + W)
        const int my_tiles = num_units > cid ? (num_units - cid + ncl - 1) / ncl : 0;
        const int total = APNN_EXP_PP == 7 ? 0 : my_tiles * nst;
        const uint32_t full0 = mapa(smem_u32(full), lead);
        if (lane == 0) {
            int ti = 0, st = 0, s = 0;
            uint32_t ph = 0;
            for (int it = 0; it < total; it++) {
                const int u = cid + ti * ncl;
                const int tm = (u % units_m) * (MC ? 2 : 1) + pic, tn = u / units_m;
                sm100::mbar_wait_sleep(&empty[s], ph ^ 1);  // parked, not spinning: the issuer needs the slots
#if APNN_EXP_PP >= 3
                if (rank == 0) mbar_arrive(&full[s]);
#else
                if (rank == 0) mbar_arrive_expect_tx(&full[s], 2u * (AST + BST));
                const uint32_t fb = full0 + (uint32_t)s * 8u;
                const int arow = (tm * 2 + (int)rank) * 128, brow = tn * BNP + (int)rank * BROWS;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    tma_load_2d_pair(sAop + (size_t)s * AST + h * AOP, &tmapA, fb, st * 256 + h * 128, arow);
                    if (!MC)
                        tma_load_2d_pair(sBop + (size_t)s * BST + h * BOP, &tmapB, fb, st * 256 + h * 128, brow);
                    else if (pic == 0)  // W half `rank` into this CTA and its counterpart in pair 1
                        tma_load_2d_pair_mc(sBop + (size_t)s * BST + h * BOP, &tmapB, fb, st * 256 + h * 128, brow,
                                            (uint16_t)((1u << rank) | (1u << (rank + 2))));
                }
#endif
                if (++st == nst) { st = 0; ti++; }
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp == PP_MMA) {
        // ------------------------------------------------------------ MMA issuer (CTA 0)
        if (rank == 0 && lane == 0) {
            const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pic));
            const uint16_t empty_mask = MC ? (uint16_t)0xF : (uint16_t)0x3;
            const uint32_t idesc = I8 ? p.idesc : idesc_mxf4(256, BNP);
            const uint32_t a0 = smem_u32(sAop), b0 = smem_u32(sBop), full_a = smem_u32(full);
            int s = 0, tc = 0, itr = 0;
            uint32_t ph = 0;
            for (int u = cid; u < num_units; u += ncl, tc++) {
                const int buf = NACC == 2 ? (tc & 1) : 0;
                mbar_wait_cluster(&accum_empty[buf], ((tc / NACC) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * BNP);
                // the next stage's barrier is probed (test_wait, non-blocking) BEFORE this stage's MMAs
                // are issued, so the probe's latency overlaps them; the blocking wait only runs when
                // the probe said "not yet" (a blocking try_wait cost ~200 cycles per stage)
                bool ready = mbar_test_wait(full_a + (uint32_t)s * 8u, ph);
                for (int st = 0; st < nst; st++, itr++) {
                    pp_tr(0, itr);
                    if (!ready && APNN_EXP_PP < 5) mbar_wait_cluster(&full[s], ph);
                    pp_tr(1, itr);
                    if (APNN_EXP_PP < 5) tc_fence_after();
                    const int s_next = s + 1 == S ? 0 : s + 1;
                    const uint32_t ph_next = s + 1 == S ? ph ^ 1 : ph;
                    ready = st + 1 < nst && mbar_test_wait(full_a + (uint32_t)s_next * 8u, ph_next);
                    const uint32_t ab = a0 + (uint32_t)s * AST, bb = b0 + (uint32_t)s * BST;
#pragma unroll
                    for (int kk = 0; kk < 8; kk++) {  // 32 bytes of K per MMA (64 e2m1 / 32 int8); boxes at AOP / BOP
                        const uint64_t da = tc::b_desc(ab + (kk >> 2) * AOP, kk & 3);
                        const uint64_t db = tc::b_desc(bb + (kk >> 2) * BOP, kk & 3);
                        if (APNN_EXP_PP == 2) continue;
                        if (I8) mma2_i8_ss(d, da, db, idesc, (st | kk) != 0);
                        else mma2_mxf4(d, da, db, idesc, tmem + SFA, tmem + SFB, (st | kk) != 0);
                    }
                    mma2_commit_mc(&empty[s], empty_mask);
                    pp_tr(2, itr);
                    s = s_next;
                    ph = ph_next;
                }
                mma2_commit_mc(&accum_full[buf], pair_mask);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;       // TMEM lane quarter
        const int slice = warp >> 2;  // column slice
        const int c_begin = slice * NCK / QW, c_end = (slice + 1) * NCK / QW;
        const int nwb = c_end - c_begin;
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t accum_empty0 = mapa(smem_u32(accum_empty), lead);
        const int ob = p.e.out_bits;
        const int Nw = (g.N + 127) / 128 * 4;
        uint8_t* stg = sStg + (size_t)warp * p.stg_warp;
        int tc = 0;
        for (int u = cid; u < num_units; u += ncl, tc++) {
            const int tm = (u % units_m) * (MC ? 2 : 1) + pic, tn = u / units_m;
            const int row0 = (tm * 2 + (int)rank) * 128 + q * 32;
            const int n0 = tn * BNP;
            if (!I32 && (p.tab_mode == tc::kTabQ3 || p.tab_mode == tc::kTabHybrid) && APNN_EXP_PP != 7) {
                named_bar_sync(1, PP_EPI * 32);  // the previous tile's table readers are done
                for (int c = threadIdx.x; c < BNP; c += PP_EPI * 32)
                    tc::build_threshold_row(sTab + c * tc::kTabStride, n0 + c, g.N, p.e);
                named_bar_sync(1, PP_EPI * 32);
            }
            const int buf = NACC == 2 ? (tc & 1) : 0;
            sm100::mbar_wait_sleep(&accum_full[buf], (uint32_t)(tc / NACC) & 1u);
            if (warp == 0 && lane == 0) pp_tr(3, tc);
            tc_fence_after();
#pragma unroll 1
            for (int c = c_begin; c < c_end && APNN_EXP_PP != 1 && APNN_EXP_PP < 4; c++) {
                uint32_t acc[32];
                tmem_ld32(tmem_lane + (uint32_t)(buf * BNP + c * 32), acc);
                tmem_wait_ld();
                if (!I8) {  // fp32 accumulator holding an exact integer
#pragma unroll
                    for (int i = 0; i < 32; i++) acc[i] = (uint32_t)__float2int_rn(__uint_as_float(acc[i]));
                }
                if (I32) {
                    // each lane writes its row's 128-byte segment (whole lines, no staging: the
                    // shared memory goes to the operand ring)
                    const int m = row0 + lane, col0 = n0 + c * 32;
                    if (m < g.M) {
                        if ((g.N & 3) == 0 && col0 + 32 <= g.N) {
                            int4* y = reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(p.Y) + (long long)m * g.N + col0);
#pragma unroll
                            for (int q4 = 0; q4 < 8; q4++)
                                y[q4] = make_int4((int)acc[4 * q4], (int)acc[4 * q4 + 1], (int)acc[4 * q4 + 2],
                                                  (int)acc[4 * q4 + 3]);
                        } else {
                            tc::epilogue_chunk(acc, m, col0, c * 32, g, p.e, p.Y, nullptr, tc::kTabNone);
                        }
                    }
                } else {
                    uint32_t w[8];
                    if (p.tab_mode == tc::kTabQ3) {
                        tc::requant_chunk_words_q3(acc, sTab, c * 32, w[0], w[1]);
                    } else {
                        tc::requant_chunk(acc, n0 + c * 32, c * 32, g, p.e, sTab, p.tab_mode, w);
                    }
                    uint32_t* srow = reinterpret_cast<uint32_t*>(stg) + lane * ob * nwb + (c - c_begin);
#pragma unroll
                    for (int tb = 0; tb < 8; tb++)
                        if (tb < ob) srow[tb * nwb] = w[tb];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(accum_empty0 + 8u * (uint32_t)buf);
            if (warp == 0 && lane == 0) pp_tr(3, 512 + tc);
            if (!I32 && row0 < g.M && APNN_EXP_PP != 1 && APNN_EXP_PP < 4) {
                __syncwarp();
                writeback_words(reinterpret_cast<const uint32_t*>(stg), lane, reinterpret_cast<uint32_t*>(p.Y), row0,
                                g.M, n0 / 32 + c_begin, Nw, ob, nwb);
            }
            __syncwarp();
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == PP_MMA) {
        tc_fence_after();
        tmem_dealloc2(tmem, 512);
    }
}

template <int BNP, bool I8>
static cudaError_t launch_pp(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid, size_t smem,
                             cudaStream_t s, bool mc) {
    auto kfn = mc ? (p.e.out_bits == 0 ? fp4_pp_kernel<BNP, true, I8, true> : fp4_pp_kernel<BNP, false, I8, true>)
                  : (p.e.out_bits == 0 ? fp4_pp_kernel<BNP, true, I8, false> : fp4_pp_kernel<BNP, false, I8, false>);
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (mc) e = cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(PP_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = mc ? 4 : 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kfn, ta, tb, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int BNP, bool AP, bool WP>
static cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid, size_t smem,
                          cudaStream_t s) {
    auto kfn = p.e.out_bits == 0 ? fp4_pair_kernel<BNP, AP, WP, true> : fp4_pair_kernel<BNP, AP, WP, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, THREADS, smem, s>>>(ta, tb, p);
    return cudaGetLastError();
}

template <int BNP>
static cudaError_t launch_enc(int enc, const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid,
                              size_t smem, cudaStream_t s) {
    switch (enc) {
    case APNN_ENC_01_01: return launch<BNP, false, false>(ta, tb, p, grid, smem, s);
    case APNN_ENC_PM1_PM1: return launch<BNP, true, true>(ta, tb, p, grid, smem, s);
    case APNN_ENC_W_PM1_A_01: return launch<BNP, false, true>(ta, tb, p, grid, smem, s);
    default: return launch<BNP, true, false>(ta, tb, p, grid, smem, s);
    }
}

}  // namespace pair
}  // namespace fp4

#if APNN_EXP_PP_TRACE
extern "C" int apnn_exp_pp_trace(unsigned long long* host, int n) {
    const int total = 8 * fp4::pair::kPpTrN;
    if (n < total) return -1;
    return cudaMemcpyFromSymbol(host, fp4::pair::g_pp_trace, total * sizeof(unsigned long long)) == cudaSuccess
               ? total : -2;
}
#endif

#if APNN_EXP_PAIR_TRACE
extern "C" int apnn_exp_pair_trace(unsigned long long* host, int n) {
    const int total = fp4::pair::TR_NEV * fp4::pair::kTrN;
    if (n < total) return -1;
    return cudaMemcpyFromSymbol(host, fp4::pair::g_trace, total * sizeof(unsigned long long)) == cudaSuccess
               ? total : -2;
}
#endif

// Pair tile width: 224 (two TMEM accumulators: epilogue overlapped) unless 256 covers the
// columns with fewer tiles; APNN_FP4_PAIR_BN (cached) forces 224 / 256 for experiments.
static int fp4_pair_bn_override() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_FP4_PAIR_BN");
        v = s ? atoi(s) : 0;
    }
    return v;
}

static const char* fp4_pair_rings() {
    static const char* v = getenv("APNN_FP4_PAIR_RINGS");
    return v;
}

int fp4_pair_pick_bn(int ncols) {
    const int o = fp4_pair_bn_override();
    if (o == 224 || o == 256) return o;
    const long long t224 = (ncols + 223) / 224, t256 = (ncols + 255) / 256;
    return t224 * 224 <= t256 * 256 + 32 ? 224 : 256;  // padded columns of the two choices
}

// prepared W (apnn_prepare_weights layout), M > 128: the persistent pair kernel
cudaError_t launch_tc_fp4_pair_prepared(const uint32_t* A, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                        int sms, cudaStream_t s) {
    using namespace fp4::pair;
    Params p;
    std::memset(&p, 0, sizeof(p));
    p.g = g;
    p.e = e;
    p.Y = Y;
    const int Kw = (g.K + 127) / 128 * 4;
    p.nst = (Kw + 7) / 8;
    p.tab_mode = tc::kTabNone;
    if (e.out_bits > 0 && e.out_bits <= 2) p.tab_mode = tc::kTabQ3;
    else if (e.out_bits > 2 && (unsigned long long)e.qmax * (unsigned long long)e.S <= 0xFFFFFFFFull)
        p.tab_mode = tc::kTabHybrid;
    p.ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;  // packed: the N padding words come out as zeros
    const int BNP = fp4_pair_pick_bn(p.ncols);
    p.tiles_m = (g.M + 255) / 256;
    p.tiles_n = (p.ncols + BNP - 1) / BNP;
    p.num_tiles = p.tiles_m * p.tiles_n;
    p.a_bytes = 32u * 128u * (uint32_t)g.a_bits;
    const int nck = BNP / 32, nwb_max = (nck + 1) / 2;
    p.stg_warp = e.out_bits == 0 ? 4096 : (32 * e.out_bits * nwb_max * 4 + 127) / 128 * 128;
    const size_t bop = (size_t)(BNP / 2) * 128;
    const size_t fixed = (size_t)EPI_WARPS * p.stg_warp + (e.out_bits ? (size_t)BNP * tc::kTabStride * 4 : 0) +
                         (2 * MAXSP + 2 * MAXS + 2 * MAXSB + 4) * 8 + 8 + DEC_WARPS * 32 * 4;
    const size_t budget = 227 * 1024 - fixed;
    // Ring depths (measured, scripts/fp4_pair_time.py, profiles/r02_fp4_pair.md): the decoded A
    // operand ring and the W ring are each refilled only after the MMA consumed the slot, so
    // both need several stages of lead (A: 4; W: the rest, it waits for an L2 round trip);
    // the A-plane ring is issued far ahead (4 = the producer's issuing lanes, its minimum).
    // APNN_FP4_PAIR_RINGS="S,SB,SP" overrides (experiments).
    int S = 4, SP = 4;
    int SB = (int)((budget - (size_t)S * AOP - (size_t)SP * p.a_bytes) / bop);
    if (SB > MAXSB) SB = MAXSB;
    if (const char* r = fp4_pair_rings()) sscanf(r, "%d,%d,%d", &S, &SB, &SP);
    // SB >= S: a decode warp waits for the W half of stage it only after the A slot of stage it
    // - S is free, so the W ring must not be lapped (the parity wait would pass on an old phase)
    // SP, SB >= kProdLanes: the producer's lanes issue kProdLanes consecutive stages in one
    // warp pass (a smaller ring would make a lane wait for a slot its own warp still has to fill)
    if (S < 2 || S > MAXS || SB < S || SB < kProdLanes || SB > MAXSB || SP < kProdLanes || SP > MAXSP)
        return cudaErrorInvalidConfiguration;
    if (SP > MAXSP) SP = MAXSP;
    if (SP < 2) return cudaErrorInvalidConfiguration;
    p.S = S;
    p.SB = SB;
    p.SP = SP;
    const size_t smem = (size_t)S * AOP + (size_t)SB * bop + (size_t)SP * p.a_bytes + fixed;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    CUtensorMap ta, tb;
    if (!fp4::make_map(&ta, A, g.M, g.a_bits, Kw, 128)) return cudaErrorInvalidValue;
    if (!fp4::make_map_prep(&tb, Wp, g.N, Kw, BNP / 2)) return cudaErrorInvalidValue;
    int pairs = sms / 2;
    if (pairs > p.num_tiles) pairs = p.num_tiles;
    const int grid = 2 * pairs;
    cudaError_t err = BNP == 224 ? launch_enc<224>(g.enc, ta, tb, p, grid, smem, s)
                                 : launch_enc<256>(g.enc, ta, tb, p, grid, smem, s);
    count_launch();
    return err;
}


// both operands prepared (apnn_gemm_prepared_ab): the persistent pair kernel without decode warps.
// Tile width: 224 (two accumulators, the epilogue overlapped with the next tile's MMAs; 8192^3
// w1a2 fused 6100 TOPS) unless APNN_FP4_PP_BN=256 (read once; one accumulator, the epilogue warps
// drain it between tiles: 5477 TOPS, scripts/fp4_pp_time.py)
static int fp4_pp_bn_override() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_FP4_PP_BN");
        v = s ? atoi(s) : 0;
    }
    return v;
}

template <int BNP, bool I32, bool I8>
static int max_clusters4(size_t smem) {
    using namespace fp4::pair;
    auto kfn = fp4_pp_kernel<BNP, I32, I8, true>;
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4);
    cfg.blockDim = dim3(PP_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kfn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

static int max_active_clusters_pp(bool i8, int bnp, bool i32, size_t smem) {
    static int cache[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
    static size_t cache_smem[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int key = (i8 ? 4 : 0) + (bnp == 224 ? 2 : 0) + (i32 ? 1 : 0);
    if (cache[key] >= 0 && cache_smem[key] == smem) return cache[key];
    int n;
    if (i8) n = i32 ? max_clusters4<256, true, true>(smem) : max_clusters4<256, false, true>(smem);
    else if (bnp == 224) n = i32 ? max_clusters4<224, true, false>(smem) : max_clusters4<224, false, false>(smem);
    else n = i32 ? max_clusters4<256, true, false>(smem) : max_clusters4<256, false, false>(smem);
    cache[key] = n;
    cache_smem[key] = smem;
    return n;
}

// both operands prepared, e2m1 (I8 = false: apnn_prepare_weights / apnn_prepare_activations rows of
// Kw * 16 bytes) or int8 (I8 = true: the _i8 preparations, rows of roundup(K, 128) bytes)
static cudaError_t launch_pp_any(const uint8_t* Ap, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y, int sms,
                                 cudaStream_t s, bool i8) {
    using namespace fp4::pair;
    Params p;
    std::memset(&p, 0, sizeof(p));
    p.g = g;
    p.e = e;
    p.Y = Y;
    const int Kw = (g.K + 127) / 128 * 4;
    const int row_bytes = i8 ? Kw * 32 : Kw * 16;
    p.nst = (row_bytes + 255) / 256;  // a stage: two 128-byte boxes of K (512 e2m1 / 256 int8 elements)
    p.tab_mode = tc::kTabNone;
    if (e.out_bits > 0 && e.out_bits <= 2) p.tab_mode = tc::kTabQ3;
    else if (e.out_bits > 2 && (unsigned long long)e.qmax * (unsigned long long)e.S <= 0xFFFFFFFFull)
        p.tab_mode = tc::kTabHybrid;
    p.ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;
    // e2m1: 224 (two accumulators beside the scale factors) unless APNN_FP4_PP_BN=256; int8: 256 with
    // two accumulators (no scale-factor columns)
    const int BNP = i8 ? 256 : (fp4_pp_bn_override() == 256 ? 256 : 224);
    p.tiles_m = (g.M + 255) / 256;
    p.tiles_n = (p.ncols + BNP - 1) / BNP;
    p.num_tiles = p.tiles_m * p.tiles_n;
    const bool a_pm1 = g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_01_A_PM1;
    const bool w_pm1 = g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_PM1_A_01;
    p.idesc = sm100::idesc_i8(256, BNP, a_pm1, w_pm1);
    const int nck = BNP / 32, nwb_max = (nck + PP_EPI / 4 - 1) / (PP_EPI / 4);
    p.stg_warp = e.out_bits == 0 ? 0 : (32 * e.out_bits * nwb_max * 4 + 127) / 128 * 128;  // int32: direct row stores
    const size_t bop = (size_t)(BNP / 2) * 128;
    const size_t fixed = (size_t)PP_EPI * p.stg_warp + (e.out_bits ? (size_t)BNP * tc::kTabStride * 4 : 0) +
                         (2 * PP_MAXS + 4) * 8 + 8;
    int S = (int)((227 * 1024 - fixed) / (2 * (AOP + bop)));
    if (S > PP_MAXS) S = PP_MAXS;
    static const int s_override = [] { const char* v = getenv("APNN_FP4_PP_STAGES"); return v ? atoi(v) : 0; }();
    if (s_override >= 2 && s_override < S) S = s_override;  // experiments: shallower rings
    if (S < 2) return cudaErrorInvalidConfiguration;
    p.S = S;
    const size_t smem = (size_t)S * 2 * (AOP + bop) + fixed;
    CUtensorMap ta, tb;
    if (!fp4::make_map_rows(&ta, Ap, g.M, row_bytes, 128)) return cudaErrorInvalidValue;
    if (!fp4::make_map_rows(&tb, Wp, g.N, row_bytes, BNP / 2)) return cudaErrorInvalidValue;
    // W multicast across the two pairs of a 4-CTA cluster (APNN_FP4_PP_MC=1, read once; off by
    // default): bit-exact and halves W's L2 -> SM bytes, but measured slower on the bench GEMM
    // (8192^3 w1a2 fused 0.203 vs 0.182 ms: fewer SMs hold whole 4-CTA clusters than CTA pairs,
    // and the two pairs advance in lockstep through the shared stage slots)
    static const int mc_env = [] { const char* v = getenv("APNN_FP4_PP_MC"); return v ? atoi(v) : 0; }();
    const bool mc = mc_env != 0 && p.tiles_m % 2 == 0 && (long long)(p.tiles_m / 2) * p.tiles_n >= sms / 4;
    int grid;
    if (mc) {
        // persistent: as many 4-CTA clusters as can be co-resident (GPC sizes need not be
        // multiples of 4), never more than the cluster units
        int clusters = max_active_clusters_pp(i8, BNP, e.out_bits == 0, smem);
        if (clusters < 1) clusters = sms / 4;
        if (clusters > (p.tiles_m / 2) * p.tiles_n) clusters = (p.tiles_m / 2) * p.tiles_n;
        grid = 4 * clusters;
    } else {
        int pairs = sms / 2;
        if (pairs > p.num_tiles) pairs = p.num_tiles;
        grid = 2 * pairs;
    }
    cudaError_t err = i8 ? launch_pp<256, true>(ta, tb, p, grid, smem, s, mc)
                         : (BNP == 224 ? launch_pp<224, false>(ta, tb, p, grid, smem, s, mc)
                                       : launch_pp<256, false>(ta, tb, p, grid, smem, s, mc));
    count_launch();
    return err;
}

cudaError_t launch_tc_fp4_pair_prepared_ab(const uint8_t* Ap, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                           int sms, cudaStream_t s) {
    return launch_pp_any(Ap, Wp, g, e, Y, sms, s, false);
}

cudaError_t launch_tc_i8_prepared_ab(const uint8_t* Ap, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                     int sms, cudaStream_t s) {
    return launch_pp_any(Ap, Wp, g, e, Y, sms, s, true);
}

}  // namespace apnn
