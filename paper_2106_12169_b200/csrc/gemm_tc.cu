// gemm_tc.cu -- tcgen05 kind::i8 variant of the AP-bit contraction (APNN_VARIANT_TC_I8).
//
// How the paper's method maps to sm_100a:
// B200 has no 1-bit tensor-core MMA (kind::b1 does not exist; the legacy b1
// mma.sync is emulated on the int8 pipe).  The paper's bit combination
//     Y = sum_s sum_t 2^(s+t) W^(s) X^(t)
// is bilinear, so it equals (sum_t 2^t X^(t)) . (sum_s 2^s W^(s))^T: the
// combination is applied to the OPERANDS (O((a+w)(M+N)K) shift-ors on the CUDA
// cores, per tile) instead of to the p.q partial products, after which one
// int8 tensor-core contraction per tile yields Y exactly.  +-1 planes decode to
// s8 -1/+1 (Cases II/III: the J terms vanish once the value
// is materialised); 0/1 codes decode to u8.
//
// Two kernels:
//   tc2_kernel (main)  persistent, CTA pair (cta_group::2): a 256 x 256 output
//                      tile per pair, M split across the two CTAs (A in each
//                      CTA's TMEM), N split across the two CTAs (B halves in
//                      each CTA's shared memory).  Warp roles per CTA:
//                        warp 0     TMA producer: one 3-D box per operand and
//                                   k-block brings ALL planes of the tile
//                                   ("virtual batching")
//                        warp 1     TMEM allocator; in CTA 0 the single-thread
//                                   tcgen05.mma issuer (4 x 256x256x32 per
//                                   k-block), int32 accumulator in TMEM
//                                   ("fragment caching")
//                        warps 2-9  recombination planes -> int8: A rows into
//                                   TMEM (tcgen05.st), B rows into the UMMA
//                                   K-major layout in smem; they run ahead into
//                                   the next tile while the epilogue drains
//                        warps 10-13 epilogue: tcgen05.ld -> int32, or the fused
//                                   element-wise routine
//   tc1_kernel         one CTA, 128 x BN tile (BN = 64/128/256), for small or
//                      skinny problems.
// K runs in blocks of 128 (the paper's b_k = 128).
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "tc_common.cuh"

namespace apnn {
namespace tc {

constexpr int BM = 128;
constexpr int T1_THREADS = 10 * 32;
constexpr int MAX_STAGES = 8;     // operand stages (A in TMEM: 32 columns each)
constexpr int MAX_PSTAGES = 16;   // packed-plane stages of the 2-CTA kernel
constexpr int kStgWarpBytes = 8192;  // store staging per epilogue warp (1024-aligned)
#ifndef APNN_PROD_LANES
#define APNN_PROD_LANES 4
#endif
constexpr int kProdLanes = APNN_PROD_LANES;  // TMA-issuing lanes of the producer warp (2-CTA kernel)
constexpr int kTunerT = 64;  // TLP threshold of the tiling heuristic (the paper's T, tuner.cu)
// Development-only knobs (pipeline trace, skipped stores / B work -- the latter two give wrong
// results by design) exist only in experiment builds: build.py --variant NAME -DAPNN_DEV=1.
#ifndef APNN_DEV
#define APNN_DEV 0
#endif
constexpr bool kDev = APNN_DEV != 0;
enum { kOutDirect = 0, kOutTma = 1, kOutLsu = 2 };

struct Params {
    Geom g;
    Epi e;
    void* Y;
    const uint32_t* A;  // raw packed activations (conv gathers rows from here)
    int stages;         // operand ring depth
    int pstages;        // plane ring depth (2-CTA kernel)
    int nkb;            // k-blocks per tile
    uint32_t a_bytes;   // A plane bytes per stage (this CTA's rows)
    uint32_t b_bytes;   // B plane bytes per stage (this CTA's rows)
    uint32_t tmem_cols;
    int tiles_m, num_tiles;
    int tab_mode;       // fused epilogue: kTabNone / kTabQ3 / kTabHybrid (tc_common.cuh)
    int out_mode;       // epilogue stores: kOutDirect / kOutTma (tensor map tmapY) / kOutLsu (coalesced)
    int nwb;            // packed TMA store box width in words (2-CTA kernel)
    int pool_fused;     // conv: 2x2/2 max pooling fused into the epilogue (pooled output Hp x Wp)
    int stg_warp;       // 2-CTA kernel: store staging bytes per epilogue warp (multiple of 1024)
    int ksplit;         // 1-CTA kernel: split-K factor Z (cluster of Z CTAs along z, DSMEM reduction)
    int Hp, Wp;
    int acc_shift;      // scaled operands: accumulator = Y << acc_shift (2-CTA kernel)
    // conv A-row tiling of the 2-CTA kernel (TMA row boxes):
    //   conv_k > 0: a CTA tile is conv_k whole output rows (conv_k * Wo <= 128 pixels)
    //   conv_k = 0: a CTA tile is a 128-pixel segment of one output row (Wo > 128)
    int conv_k, conv_bw, conv_segs, conv_nbox;
    int conv_box_stride;  // bytes between row boxes in a plane stage (16*bw*bits rounded up to 128: TMA dst alignment)
    int conv_merged;      // C_in <= 128: a pixel's planes are one contiguous record, fetched as ONE box row
                          // ({4*bits words, pixels} box, smem [pixel][plane][16 B]) instead of bits rows
    uint32_t a_tx_bytes;  // bytes the A loads of one stage actually deliver (expect_tx; excludes slot padding)
    unsigned long long* trace;  // development trace (APNN_TRACE), nullptr normally
    int exp_nostore;            // experiment knob (APNN_EXP_NOSTORE): skip the epilogue stores
    int exp_nob;                // experiment knob (APNN_EXP_NOB): B warps skip the decode (wrong results)
    int halves;                 // 256-wide pair tiles: two N = 128 MMA halves (APNN_HALVES, default 0)
    int prep;                   // prepared int8 W (apnn_prepare_weights_i8): B tiles by TMA, no B decode
};

// development trace of CTA 0: clock64 stamps per k-block / tile (APNN_TRACE=<file>)
constexpr int kTraceN = 2048;
enum { TR_PROD = 0, TR_A_PLANE = 1, TR_A_OP = 2, TR_A_DONE = 3, TR_MMA_OPFULL = 4, TR_MMA_ISSUED = 5,
       TR_EPI_FULL = 6, TR_EPI_DONE = 7, TR_N = 8 };
__device__ __forceinline__ void trace_at(const Params& p, int ev, int idx) {
    if (kDev && p.trace && blockIdx.x == 0 && idx < kTraceN) {
        unsigned long long c;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
        p.trace[ev * kTraceN + idx] = c;
    }
}
// per-CTA %globaltimer stamps (ns): 0 entry, 1 after the prologue, 2 work done, 3 exit
constexpr int kCtaTraceMax = 1024;
// CTA-0 event stamps (ns), slots 0..31 (development)
__device__ __forceinline__ void dbg_stamp(const Params& p, int slot) {
    if (kDev && p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[kTraceN * TR_N + 4 * kCtaTraceMax + slot] = t;
    }
}
__device__ __forceinline__ void cta_stamp(const Params& p, int k) {
    const int b = blockIdx.x + (blockIdx.y + blockIdx.z * gridDim.y) * gridDim.x;
    if (kDev && p.trace && threadIdx.x == 0 && b < kCtaTraceMax) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[kTraceN * TR_N + b * 4 + k] = t;
    }
}

// Rows of CTA tile `ct`: output rows m_base .. m_base + len - 1 (GEMM: 128-row tiles).
__device__ __forceinline__ void cta_tile_rows(const Params& p, int ct, int& m_base, int& len) {
    const Geom& g = p.g;
    if (!g.conv) {
        m_base = ct * 128;
        len = 128;
    } else if (p.conv_k > 0) {
        m_base = ct * p.conv_k * g.Wo;
        len = p.conv_k * g.Wo;
    } else {
        const int gr = ct / p.conv_segs, sg = ct - gr * p.conv_segs;
        m_base = gr * g.Wo + sg * 128;
        len = min(128, g.Wo - sg * 128);
    }
    if (m_base + len > g.M) len = g.M - m_base;
    if (len < 0) len = 0;
}

__device__ __forceinline__ void tma_load_2d_box(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(sm100::smem_u32(dst)),
        "l"(tmap), "r"(sm100::smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// ------------------------------------------------- fused 2x2/2 max pooling
// (fused conv + pool + quantisation 641-647).  q is non-decreasing in
// v = alpha*y + beta, so the max over a grid of q equals q of the max v (reading R15):
// every row (output pixel) requantises its own 32 channels, the four codes of a 2x2
// grid are combined with a byte-wise max through shared memory, and the grid's
// top-left pixel ("anchor") packs and stores the pooled codes.  The CTA tile holds
// conv_k (even) whole output rows and Ho is even, so every grid lies in one tile.
__device__ __forceinline__ bool pool_anchor(int t, int len, int mb, const Geom& g, const Params& p, long long& prow) {
    if (t >= len) return false;
    const int i = t / g.Wo, wo = t - i * g.Wo;
    if ((i & 1) || (wo & 1) || wo + 1 >= g.Wo) return false;
    const int gr = mb / g.Wo + i;          // global output row b*Ho + ho (ho even)
    const int b = gr / g.Ho, ho = gr - b * g.Ho;
    prow = ((long long)b * p.Hp + (ho >> 1)) * p.Wp + (wo >> 1);
    return true;
}

__device__ __forceinline__ void pool_chunk(const uint32_t (&acc)[32], int nb, int lc, int t, int len, int mb,
                                           const Geom& g, const Params& p, const int32_t* tab, uint8_t* buf) {
    uint32_t qb[8];
    requant_chunk_bytes(acc, nb, lc, g, p.e, tab, p.tab_mode, qb);
    uint4* row = reinterpret_cast<uint4*>(buf + t * 32);
    row[0] = make_uint4(qb[0], qb[1], qb[2], qb[3]);
    row[1] = make_uint4(qb[4], qb[5], qb[6], qb[7]);
    sm100::named_bar_sync(2, 128);
    long long prow;
    if (!pool_anchor(t, len, mb, g, p, prow)) return;
    const int nbrs[3] = {t + 1, t + g.Wo, t + g.Wo + 1};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const uint4* r = reinterpret_cast<const uint4*>(buf + nbrs[k] * 32);
        const uint4 a = r[0], b = r[1];
        qb[0] = __vmaxu4(qb[0], a.x); qb[1] = __vmaxu4(qb[1], a.y);
        qb[2] = __vmaxu4(qb[2], a.z); qb[3] = __vmaxu4(qb[3], a.w);
        qb[4] = __vmaxu4(qb[4], b.x); qb[5] = __vmaxu4(qb[5], b.y);
        qb[6] = __vmaxu4(qb[6], b.z); qb[7] = __vmaxu4(qb[7], b.w);
    }
    const int Nw = (g.N + 127) / 128 * 4;
    if (nb / 32 >= Nw) return;  // chunk entirely in the last tile's overhang past the N padding
    uint32_t w[8];
    bytes_to_words(qb, p.e.out_bits, w);
    uint32_t* o = reinterpret_cast<uint32_t*>(p.Y) + prow * p.e.out_bits * Nw + nb / 32;
#pragma unroll
    for (int tb = 0; tb < 8; tb++)
        if (tb < p.e.out_bits) o[(long long)tb * Nw] = w[tb];
}

// zero the N padding words [w_from, Nw) of the pooled rows anchored in this tile
__device__ __forceinline__ void pool_pad_words(int n_end, int t, int len, int mb, const Geom& g, const Params& p) {
    const int Nw = (g.N + 127) / 128 * 4;
    if (n_end < g.N) return;
    long long prow;
    if (!pool_anchor(t, len, mb, g, p, prow)) return;
    uint32_t* o = reinterpret_cast<uint32_t*>(p.Y) + prow * p.e.out_bits * Nw;
    for (int tb = 0; tb < p.e.out_bits; tb++)
        for (int w = n_end / 32; w < Nw; w++) o[(long long)tb * Nw + w] = 0u;
}

// ============================================================== 2-CTA kernel
// Warp roles.  The warp scheduler arbitrates highest-warp-id first (B300_MICROARCH.md),
// so the single-thread MMA issuer and the TMA producer get the highest ids.
constexpr int T2_RECOMB_WARPS = 16;                 // warps 0-15: two teams of 8 on alternating k-blocks
constexpr int T2_EPI0 = T2_RECOMB_WARPS;            // warps 16-19: epilogue
constexpr int T2_TMA_WARP = T2_EPI0 + 4;            // warp 20: TMA producer / conv gather
constexpr int T2_MMA_WARP = T2_TMA_WARP + 1;        // warp 21: TMEM allocator + MMA issuer (CTA 0)
constexpr int T2_THREADS = (T2_MMA_WARP + 1) * 32;

// BNP = N of the pair tile (256 / 128 / 64); each CTA holds BNP/2 B rows.
template <int BNP, bool A_PM1, bool W_PM1, bool SCALED, bool RES = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1)
    tc2_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
               const __grid_constant__ CUtensorMap tmapY, const Params p) {
    using namespace sm100;
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int BROWS = BNP / 2;                               // B rows per CTA
    constexpr int T2_BN = BNP;
    constexpr uint32_t BOP_STAGE = BROWS * 128;                  // bytes of one B operand stage
    const int S = p.stages, SP = p.pstages;
    uint8_t* sBop = smem;                                        // S x BROWS rows x 128 B
    uint8_t* sStg = sBop + (size_t)S * BOP_STAGE;                // 4 epilogue warps x 8 KB TMA-store staging
    uint8_t* sApl = sStg + 4 * p.stg_warp;                       // SP x a_bytes
    uint8_t* sBpl = sApl + (size_t)SP * p.a_bytes;               // SP x b_bytes
    int32_t* sTab = reinterpret_cast<int32_t*>(sBpl + (size_t)SP * p.b_bytes);  // 256 x 16 int32
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + T2_BN * kTabStride);
    uint64_t* plane_full = bars;                                   // [MAX_PSTAGES]
    uint64_t* plane_empty = bars + MAX_PSTAGES;                    // [MAX_PSTAGES]
    uint64_t* op_full = bars + 2 * MAX_PSTAGES;                    // [MAX_STAGES], used in CTA 0
    uint64_t* op_empty = op_full + MAX_STAGES;                     // [MAX_STAGES]
    // accumulators: NACC = 2 TMEM buffers when the pair tile is <= 128 columns wide (the
    // epilogue of tile i then overlaps the MMAs of tile i+1), else 1 (A stages fill the rest)
    constexpr int NACC = T2_BN <= 128 ? 2 : 1;
    // 256-wide tiles: the MMA runs as two N = 128 halves (accumulator columns [0,128) and
    // [128,256), B rows [0,64) / [64,128) of each CTA), released separately by the epilogue,
    // so the next tile's first MMAs start after half the epilogue.  Experiment only
    // (APNN_HALVES=1): the N = 128 instructions made the main loop slower than the exposure saved
    constexpr bool HALVES = T2_BN == 256;
    uint64_t* accum_full = op_empty + MAX_STAGES;                  // [2]
    uint64_t* accum_empty = accum_full + 2;                        // [2], used in CTA 0
    uint64_t* b_full = accum_empty + 2;                            // [MAX_STAGES] prepared W landed (p.prep)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(b_full + MAX_STAGES);
    volatile uint32_t* dep_slots = tmem_holder + 1;                // [T2_RECOMB_WARPS * 32]

    cta_stamp(p, 0);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const Geom& g = p.g;
    const int nkb = p.nkb;

    if (warp == T2_TMA_WARP && lane == 0) {
        tma_prefetch(&tmapA);
        tma_prefetch(&tmapB);
        if (p.out_mode == kOutTma) tma_prefetch(&tmapY);
        for (int s = 0; s < SP; s++) {
            mbar_init(&plane_full[s], 1);
            mbar_init(&plane_empty[s], 8);
        }
        for (int s = 0; s < S; s++) {
            mbar_init(&op_full[s], 16);   // 8 recombination warps x 2 CTAs
            mbar_init(&op_empty[s], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&accum_full[i], 1);
            mbar_init(&accum_empty[i], 8);  // 4 epilogue warps x 2 CTAs
        }
        for (int i = 0; i < S; i++) mbar_init(&b_full[i], 1);
        fence_mbar_init();
    }
    if (warp == T2_MMA_WARP) tmem_alloc2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    constexpr uint32_t A_COL = 256;
    cta_stamp(p, 1);

    if (warp == T2_TMA_WARP) {
        // ---------------------------------------------------- TMA producer
        // (conv: one strided TMA box per output row of the tile and filter tap;
        //  out-of-frame pixels are zero-filled by the TMA unit)
        // Lanes 0..kProdLanes-1 issue consecutive k-blocks side by side: one warp
        // instruction carries kProdLanes expect_tx arrivals and box loads, which hides
        // the ~200-cycle per-stage barrier round trip of a single issuing thread
        // (scripts/tma_rate.cu: 330 -> 137 cycles per 128-row box with 4 lanes; the TMA
        // unit then runs at about one 16-byte box row per cycle).
        const bool conv = g.conv;
        const int my_tiles = p.num_tiles > cid ? (p.num_tiles - cid + ncl - 1) / ncl : 0;
        const int total = my_tiles * nkb;
        for (int base = 0; base < total; base += kProdLanes) {
            const int it = base + lane;
            if (lane < kProdLanes && it < total) {
                const int s = it % SP;
                const uint32_t ph = (uint32_t)(it / SP) & 1u;
                const int ti = it / nkb, kb = it - ti * nkb;
                const int tile = cid + ti * ncl;
                const int ct = (tile % p.tiles_m) * 2 + rank;
                const int m0 = ct * 128;
                const int nr0 = (tile / p.tiles_m) * T2_BN + rank * BROWS;
                mbar_wait(&plane_empty[s], ph ^ 1);
                if (lane == 0) trace_at(p, TR_PROD, it);
                const int rs = conv ? kb / g.CB : 0;
                const int cb = conv ? kb - rs * g.CB : kb;
                mbar_arrive_expect_tx(&plane_full[s], p.a_tx_bytes + (p.prep ? 0u : p.b_bytes));
                uint8_t* adst = sApl + (size_t)s * p.a_bytes;
                if (!conv) {
                    tma_load_4d(adst, &tmapA, &plane_full[s], kb * 4, m0, 0, 0);
                } else {
                    const int r = rs / g.S, sx = rs - r * g.S;
                    const int box_bytes = p.conv_box_stride;
                    for (int i = 0; i < p.conv_nbox; i++) {
                        int gr, wo0;
                        if (p.conv_k > 0) { gr = ct * p.conv_k + i; wo0 = 0; }
                        else { gr = ct / p.conv_segs; wo0 = (ct - gr * p.conv_segs) * 128; }
                        const int b = gr / g.Ho, ho = gr - b * g.Ho;  // b >= B -> whole box out of bounds (zeros)
                        if (p.conv_merged)
                            tma_load_4d(adst + i * box_bytes, &tmapA, &plane_full[s], 0, wo0 * g.stride + sx - g.pad,
                                        ho * g.stride + r - g.pad, b);
                        else
                            tma_load_5d(adst + i * box_bytes, &tmapA, &plane_full[s], cb * 4,
                                        wo0 * g.stride + sx - g.pad, 0, ho * g.stride + r - g.pad, b);
                    }
                }
                if (!p.prep) {
                    tma_load_4d(sBpl + (size_t)s * p.b_bytes, &tmapB, &plane_full[s], cb * 4, nr0, 0, rs);
                } else {  // prepared int8 W (GEMM): 128 bytes x BROWS rows straight into operand stage os
                    const int os = it % S;
                    const uint32_t oph = (uint32_t)(it / S) & 1u;
                    mbar_wait(&op_empty[os], oph ^ 1);
                    mbar_arrive_expect_tx(&b_full[os], BOP_STAGE);
                    tma_load_2d_box(sBop + (size_t)os * BOP_STAGE, &tmapB, &b_full[os], kb * 128, nr0);
                }
            }
            __syncwarp();
        }
    } else if (warp == T2_MMA_WARP) {
        // ---------------------------------------------------- MMA issuer (CTA 0)
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = idesc_i8(256, (HALVES && p.halves) ? 128 : T2_BN, A_PM1, W_PM1);
            const uint64_t bdesc0 = b_desc(smem_u32(sBop), 0);
            const uint32_t a_col0 = tmem + A_COL;
            int s = 0, tc = 0;
            uint32_t ph = 0;
            for (int tile = cid; tile < p.num_tiles; tile += ncl, tc++) {
                const int buf = tc % NACC;
                const uint32_t dtm = tmem + (uint32_t)(buf * T2_BN);
                const bool halves = HALVES && p.halves;
                mbar_wait_cluster(&accum_empty[buf], ((tc / NACC) & 1) ^ 1);  // halves: the low half
                tc_fence_after();
                for (int kb = 0; kb < nkb; kb++) {
                    mbar_wait_cluster(&op_full[s], ph);
                    trace_at(p, TR_MMA_OPFULL, tc * nkb + kb);
                    tc_fence_after();
                    const uint64_t bd = bdesc0 + (uint64_t)(s * (BOP_STAGE / 16));
                    const uint32_t as = a_col0 + s * 32;
                    if (!halves) {
#pragma unroll
                        for (int kk = 0; kk < 4; kk++)
                            mma2_i8_ts(dtm, as + kk * 8, bd + (uint64_t)(kk * kBDescKStep), idesc, (kb | kk) != 0);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < 4; kk++)
                            mma2_i8_ts(dtm, as + kk * 8, bd + (uint64_t)(kk * kBDescKStep), idesc, (kb | kk) != 0);
                        if (kb == 0) {  // the high half of the accumulator must be drained too
                            mbar_wait_cluster(&accum_empty[1], (tc & 1) ^ 1);
                            tc_fence_after();
                        }
                        const uint64_t bdh = bd + (uint64_t)(64 * 128 / 16);  // B rows 64..127 of each CTA
#pragma unroll
                        for (int kk = 0; kk < 4; kk++)
                            mma2_i8_ts(dtm + 128, as + kk * 8, bdh + (uint64_t)(kk * kBDescKStep), idesc,
                                       (kb | kk) != 0);
                    }
                    mma2_commit_mc(&op_empty[s], 0x3);
                    trace_at(p, TR_MMA_ISSUED, tc * nkb + kb);
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                mma2_commit_mc(&accum_full[buf], 0x3);
            }
        }
    } else if (warp < T2_EPI0) {
        // ---------------------------------------------------- recombination
        // team (0/1) handles k-blocks of its parity, so two k-blocks are in flight
        // per SM sub-partition; inside a team warps 0-3 decode A rows, 4-7 B rows.
        const int q = warp & 3;
        const int team = warp >> 3;
        const int grp = (warp >> 2) & 1;
        const int t = q * 32 + lane;
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t op_full0 = mapa(smem_u32(op_full), 0);
        int it = 0, s = 0, ps = 0;
        uint32_t ph = 0, pph = 0;
        // A job source row inside the plane stage: conv stages hold conv_nbox row boxes
        // of conv_bw pixels ([box][plane][pixel][16 B]); unused tile rows read row 0
        int a_box = 0, a_row = t, a_rows = 128;
        if (g.conv) {
            const int tt = t < p.conv_nbox * p.conv_bw ? t : 0;
            a_box = tt / p.conv_bw;
            a_row = tt - a_box * p.conv_bw;
            a_rows = p.conv_bw;
        }
        const uint32_t a_box_off = (uint32_t)(a_box * p.conv_box_stride);
        for (int tile = cid; tile < p.num_tiles; tile += ncl) {
            RowCtx rc;
            if (A_PM1 && g.conv) {
                int mb, len;
                cta_tile_rows(p, (tile % p.tiles_m) * 2 + rank, mb, len);
                rc = make_row(g, t < len ? mb + t : g.M);
            }
            for (int kb = 0; kb < nkb; kb++, it++, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0),
                     ps = (ps + 1 == SP) ? 0 : ps + 1, pph ^= (ps == 0)) {
                if ((it & 1) != team) continue;
                int kvalid = 128;  // +-1 activations: elements beyond kvalid decode to 0
                if (A_PM1) {
                    if (g.conv) {
                        kvalid = conv_kvalid(g, rc, kb_tap(g, kb));
                    } else if (W_PM1) {
                        const int rem = g.K - kb * 128;
                        kvalid = rem < 128 ? rem : 128;
                    }
                }
                mbar_wait(&plane_full[ps], pph);
                if (warp == 0 && lane == 0) trace_at(p, TR_A_PLANE, it >> 1);
                if (grp == 0) {
                    recomb_step_any<A_PM1, true, SCALED>(g.a_bits, sApl + (size_t)ps * p.a_bytes + a_box_off,
                                                         p.conv_merged ? 1 : a_rows, p.conv_merged ? g.a_bits : 1,
                                                         a_row, &plane_empty[ps],
                                                 &op_empty[s], ph ^ 1, tmem_lane + A_COL + s * 32, nullptr, kvalid,
                                                 lane, dep_slots + threadIdx.x);
                    tmem_wait_st();
                } else if (p.prep) {  // prepared W: the B tile comes from TMA; keep the barrier protocol
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&plane_empty[ps]);
                    mbar_wait(&b_full[s], ph);
                } else if (t < BROWS && !(kDev && p.exp_nob)) {  // warp-uniform: BROWS is a multiple of 32
                    recomb_step_any<W_PM1, false, SCALED>(g.w_bits, sBpl + (size_t)ps * p.b_bytes, BROWS, 1, t,
                                                          &plane_empty[ps], &op_empty[s], ph ^ 1, 0,
                                                          sBop + (size_t)s * BOP_STAGE, 128, lane,
                                                          dep_slots + threadIdx.x);
                    fence_proxy_async_smem();
                } else {                 // idle B warp (narrow pair tile): nothing to write, but it
                    // must keep the barrier phase accounting of a writer: release the plane
                    // stage, and wait for the previous use of the operand stage to be consumed
                    // before arriving on op_full (an early arrival would complete the
                    // previous use's phase before the real writers finish -- measured as a
                    // rare wrong k-block).
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&plane_empty[ps]);
                    mbar_wait(&op_empty[s], ph ^ 1);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(op_full0 + s * 8);
                if (warp == 0 && lane == 0) trace_at(p, TR_A_DONE, it >> 1);
            }
        }
    } else {
        // ---------------------------------------------------- epilogue
        // Each warp owns 32 rows of the CTA tile (its TMEM lane quarter).  Stores go
        // through shared-memory staging and TMA (coalesced, clipped at M / N): int32
        // as 32 x 32 swizzled blocks (double-buffered per warp), packed codes as one
        // {nwb words, out_bits, 32 rows} box per tile.  Warps whose 32-row slab runs
        // past a conv tile's rows store directly (the box would overwrite the next
        // tile's rows).
        const int q = warp & 3;
        const int t = q * 32 + lane;               // row in this CTA's 128
        const int et = threadIdx.x - T2_EPI0 * 32;  // 0..127
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t accum_empty0 = mapa(smem_u32(accum_empty), 0);  // + 8 * buf
        const int ob = p.e.out_bits;
        uint8_t* stg = sStg + q * p.stg_warp;
        const uint32_t stg_addr = smem_u32(stg);
        int tc = 0;
        uint32_t nst = 0, npc = 0;
        for (int tile = cid; tile < p.num_tiles; tile += ncl, tc++) {
            int mb, len;
            cta_tile_rows(p, (tile % p.tiles_m) * 2 + rank, mb, len);
            const int m = t < len ? mb + t : g.M;   // rows beyond the tile are not stored
            const int n0 = (tile / p.tiles_m) * T2_BN;
            const bool any = q * 32 < len;
            const bool use_tma = p.out_mode == kOutTma && any && (!g.conv || q * 32 + 32 <= len) && !(kDev && p.exp_nostore);
            const bool use_lsu = p.out_mode == kOutLsu && any && !(kDev && p.exp_nostore);
            const int row0 = mb + q * 32, row_end = mb + len;
            if (p.tab_mode == kTabQ3 || p.tab_mode == kTabHybrid) {
                named_bar_sync(1, 128);  // previous tile's readers are done
                if (et < T2_BN) build_threshold_row(sTab + et * kTabStride, n0 + et, g.N, p.e);
                if (et + 128 < T2_BN) build_threshold_row(sTab + (et + 128) * kTabStride, n0 + et + 128, g.N, p.e);
                named_bar_sync(1, 128);
            }
            if (ob && use_tma) {  // the previous tile's packed box has been read out of staging
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
            }
            const int buf = tc % NACC;
            mbar_wait(&accum_full[buf], (tc / NACC) & 1);
            if (warp == T2_EPI0 && lane == 0) trace_at(p, TR_EPI_FULL, tc);
            tc_fence_after();
            const bool halves = HALVES && p.halves;
#pragma unroll 1
            for (int cc = 0; cc < T2_BN; cc += 32) {
                uint32_t acc[32];
                tmem_ld32(tmem_lane + (uint32_t)(buf * T2_BN) + cc, acc);
                tmem_wait_ld();
                // accumulator column cc -> tile-local output column c (halves: [0,64) CTA0 B rows
                // 0-63, [64,128) CTA1 rows 0-63, [128,192) CTA0 rows 64-127, [192,256) CTA1 rows 64-127)
                int c = cc;
                if (halves) {
                    const int h = cc >> 7, j = cc & 127;
                    c = j < 64 ? 64 * h + j : 128 + 64 * h + (j - 64);
                    if (cc == 96) {  // the low half has been read out: release it to the next tile
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(accum_empty0);
                    }
                }
                if (SCALED) {
#pragma unroll
                    for (int i = 0; i < 32; i++) acc[i] = (uint32_t)((int32_t)acc[i] >> p.acc_shift);
                }
                if (p.pool_fused) {  // uniform across the 4 epilogue warps (named barrier inside)
                    pool_chunk(acc, n0 + c, c, t, len, mb, g, p, sTab, sStg + (npc & 1) * 4096);
                    __syncwarp();  // reconverge before the next .sync.aligned TMEM load
                    npc++;
                    continue;
                }
                if (!any || (kDev && p.exp_nostore)) continue;
                if (ob == 0) {
                    if (use_tma) {
                        uint8_t* b = stg + (nst & 1) * 4096;
                        if (lane == 0) bulk_wait_read<1>();  // this buffer's store (two ago) has been read
                        __syncwarp();
                        stage_int32_chunk(acc, b, lane);
                        fence_async_smem_cta();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmapY, smem_u32(b), n0 + c, mb + q * 32);
                            bulk_commit();
                        }
                        nst++;
                    } else if (use_lsu) {
                        stage_int32_chunk(acc, stg, lane);
                        __syncwarp();
                        writeback_int32_block(stg, lane, reinterpret_cast<int32_t*>(p.Y), row0, row_end, n0 + c, g.N);
                        __syncwarp();
                    } else {
                        epilogue_chunk(acc, m, n0 + c, c, g, p.e, p.Y, nullptr, kTabNone);
                    }
                } else if (use_tma || use_lsu) {
                    uint32_t w[8];
                    requant_chunk<RES>(acc, n0 + c, c, g, p.e, sTab, p.tab_mode, w, m);
                    stage_words(w, ob, p.nwb, c >> 5, reinterpret_cast<uint32_t*>(stg), lane);
                } else {
                    epilogue_chunk<RES>(acc, m, n0 + c, c, g, p.e, p.Y, sTab, p.tab_mode);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(accum_empty0 + 8u * (uint32_t)(halves ? 1 : buf));
            if (p.pool_fused) {
                pool_pad_words(n0 + T2_BN, t, len, mb, g, p);
            } else if (ob && any && !(kDev && p.exp_nostore)) {
                if (use_tma || use_lsu) {
                    const uint32_t zero8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    for (int wi = T2_BN / 32; wi < p.nwb; wi++)  // box words past the tile: N padding
                        stage_words(zero8, ob, p.nwb, wi, reinterpret_cast<uint32_t*>(stg), lane);
                }
                if (use_tma) {
                    fence_async_smem_cta();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&tmapY, stg_addr, n0 / 32, 0, row0);
                        bulk_commit();
                    }
                } else if (use_lsu) {
                    __syncwarp();
                    writeback_packed_block(reinterpret_cast<const uint32_t*>(stg), lane, reinterpret_cast<uint32_t*>(p.Y),
                                           row0, row_end, n0 / 32, (g.N + 127) / 128 * 4, ob, p.nwb);
                    __syncwarp();
                } else if (n0 + T2_BN >= g.N) {
                    zero_pad_words(m, (n0 + T2_BN) / 32, g, p.e, p.Y);
                }
            }
            if (warp == T2_EPI0 && lane == 0) trace_at(p, TR_EPI_DONE, tc);
        }
        if (lane == 0) bulk_wait<0>();
    }

    tc_fence_before();
    __syncthreads();
    cta_stamp(p, 2);
    cluster_sync();
    if (warp == T2_MMA_WARP) {
        tc_fence_after();
        tmem_dealloc2(tmem, p.tmem_cols);
    }
    cta_stamp(p, 3);
}

// ------------------------------------------------ split-K reduction (row f4)
// Small problems (few output tiles) leave most SMs idle.  The 1-CTA kernel then runs
// Z = ksplit CTAs per output tile as one thread-block cluster along z; CTA z reduces
// k-blocks [z*nkb/Z, (z+1)*nkb/Z).  Each CTA parks its 128 x BN int32 partial sums in
// a reduction region of its own shared memory (16-byte chunks XOR-swizzled by row:
// conflict-free row-per-thread stores), the cluster synchronises, and CTA z sums rows
// [z*128/Z, (z+1)*128/Z) over all Z partials through distributed shared memory
// (ld.shared::cluster, all Z loads in flight; measured faster than pushing the
// partials with st.shared::cluster), then applies the epilogue: one warp per (row, 32-column chunk), lane = column, so int32
// stores are coalesced and packed words come from __ballot_sync.
__device__ __forceinline__ int split_red_index(int row, int col, int BN) {
    return row * BN + ((((col >> 2) ^ (row & 7))) << 2) + (col & 3);
}
__device__ __forceinline__ int32_t ld_cluster_s32(uint32_t cluster_addr) {
    int32_t v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(cluster_addr));
    return v;
}

template <int BN>
__device__ __forceinline__ void split_reduce_store(const Params& p, uint8_t* smem, int m0, int n0,
                                                   const int32_t* tab, int warp, int lane) {
    using namespace sm100;
    const Geom& g = p.g;
    const int Z = p.ksplit;
    const uint32_t z = cluster_ctarank();
    if (threadIdx.x == 64) dbg_stamp(p, 4);
    cluster_sync();  // every partial of the cluster is in shared memory
    if (threadIdx.x == 64) dbg_stamp(p, 5);
    const uint32_t red0 = smem_u32(smem);
    const int rows = BM / Z;
    const int nch = BN / 32;
    const int units = rows * nch;
    const int ob = p.e.out_bits;
    const int Nw = (g.N + 127) / 128 * 4;
    for (int u = warp; u < units; u += T1_THREADS / 32) {
        const int row = (int)z * rows + u / nch, ch = u - (u / nch) * nch;
        const int col = ch * 32 + lane;
        const uint32_t off = red0 + 4u * (uint32_t)split_red_index(row, col, BN);
        int32_t part[8];  // all Z remote loads in flight before the sum
#pragma unroll
        for (int r = 0; r < 8; r++) part[r] = r < Z ? ld_cluster_s32(mapa(off, (uint32_t)r)) : 0;
        int32_t y = 0;
#pragma unroll
        for (int r = 0; r < 8; r++) y += part[r];
        const int m = m0 + row, n = n0 + col;
        if (m >= g.M) continue;  // warp-uniform
        if (ob == 0) {
            if (n < g.N) reinterpret_cast<int32_t*>(p.Y)[(long long)m * g.N + n] = y;
        } else {
            uint32_t q = 0;
            if (n < g.N) {
                if (p.tab_mode == kTabQ3) {
                    const int4 h = *reinterpret_cast<const int4*>(tab + col * kTabStride);
                    const int32_t yp = y * h.x;
                    q = (uint32_t)(yp > h.y) + (uint32_t)(yp > h.z) + (uint32_t)(yp > h.w);
                } else if (p.tab_mode == kTabHybrid) {
                    q = requant_hybrid(tab + col * kTabStride, y, (uint32_t)p.e.S, p.e.invS, (uint32_t)p.e.qmax);
                } else {
                    q = requant(p.e, y, epi_alpha(p.e, n), epi_beta(p.e, n));
                }
            }
            const int word = (n0 >> 5) + ch;
            uint32_t* o = reinterpret_cast<uint32_t*>(p.Y) + (long long)m * ob * Nw + word;
            for (int tb = 0; tb < ob; tb++) {
                const uint32_t wv = __ballot_sync(0xFFFFFFFFu, (q >> tb) & 1u);
                if (lane == tb && word < Nw) o[(long long)tb * Nw] = wv;
            }
        }
    }
    if (threadIdx.x == 64) dbg_stamp(p, 6);
    cluster_sync();  // remote reads done before any CTA of the cluster exits
}

// ============================================================== 1-CTA kernel

template <int BN, bool A_PM1, bool W_PM1>
__global__ void __launch_bounds__(T1_THREADS, 1)
    tc1_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
               const __grid_constant__ CUtensorMap tmapY, const Params p) {
    using namespace sm100;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    // split-K: a dedicated reduction region first (other CTAs of the cluster push into it
    // while this CTA may still be in its main loop), then the pipeline buffers
    uint8_t* sBop = smem + (p.ksplit > 1 ? BM * BN * 4 : 0);  // S x BN x 128 B
    uint8_t* sApl = sBop + (size_t)S * BN * 128;             // S x a_bytes
    uint8_t* sBpl = sApl + (size_t)S * p.a_bytes;            // S x b_bytes
    int32_t* sTab = reinterpret_cast<int32_t*>(sBpl + (size_t)S * p.b_bytes);  // BN x 16 int32
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + BN * kTabStride);
    uint64_t* plane_full = bars;
    uint64_t* plane_empty = bars + MAX_STAGES;
    uint64_t* op_full = bars + 2 * MAX_STAGES;
    uint64_t* op_empty = bars + 3 * MAX_STAGES;
    uint64_t* accum_full = bars + 4 * MAX_STAGES;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * MAX_STAGES + 2);

    cta_stamp(p, 0);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const Geom& g = p.g;
    // split-K (f4, small problems): CTA z of the cluster reduces k-blocks [kb0, kb0 + nkb)
    const int kb0 = (int)(((long long)blockIdx.z * p.nkb) / p.ksplit);
    const int nkb = (int)(((long long)(blockIdx.z + 1) * p.nkb) / p.ksplit) - kb0;  // >= 1 (ksplit <= nkb)

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmapA);
        tma_prefetch(&tmapB);
        for (int s = 0; s < S; s++) {
            mbar_init(&plane_full[s], g.conv ? 1 + 32 : 1);
            mbar_init(&plane_empty[s], 8);
            mbar_init(&op_full[s], 8);
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
    constexpr uint32_t A_COL = BN;
    cta_stamp(p, 1);

    if (warp == 0) {
        const bool conv = g.conv;
        if (conv || lane == 0) {
            RowCtx rc[4];
            if (conv) {
#pragma unroll
                for (int i = 0; i < 4; i++) rc[i] = make_row(g, m0 + lane + 32 * i);
            }
            for (int i = 0; i < nkb; i++) {
                const int kb = kb0 + i;
                const int s = i % S;
                const uint32_t ph = (i / S) & 1;
                mbar_wait(&plane_empty[s], ph ^ 1);
                if (lane == 0) {
                    const int rs = conv ? kb / g.CB : 0;
                    const int cb = conv ? kb - rs * g.CB : kb;
                    mbar_arrive_expect_tx(&plane_full[s], (conv ? 0u : p.a_bytes) + p.b_bytes);
                    if (i == 0) dbg_stamp(p, 0);
                    if (!conv) tma_load_4d(sApl + (size_t)s * p.a_bytes, &tmapA, &plane_full[s], kb * 4, m0, 0, 0);
                    tma_load_4d(sBpl + (size_t)s * p.b_bytes, &tmapB, &plane_full[s], cb * 4, n0, 0, rs);
                }
                if (conv) conv_gather_kb<4>(p.A, g, rc, kb, sApl + (size_t)s * p.a_bytes, BM, lane, &plane_full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(BM, BN, A_PM1, W_PM1);
            for (int kb = 0; kb < nkb; kb++) {  // local k-block index
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&op_full[s], ph);
                tc_fence_after();
                const uint32_t bbase = smem_u32(sBop + (size_t)s * BN * 128);
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    const uint64_t bdesc = b_desc(bbase, kk);
                    mma_i8_ts(tmem, tmem + A_COL + s * 32 + kk * 8, bdesc, idesc, (kb | kk) != 0);
                }
                mma_commit(&op_empty[s]);
            }
            mma_commit(accum_full);
        }
    } else {
        const int q = warp & 3;
        const int grp = (warp - 2) >> 2;
        const int t = q * 32 + lane;
        const int et = threadIdx.x - 64;  // 0..255
        const uint32_t tmem_lane = tmem + ((uint32_t)(q * 32) << 16);
        if ((p.tab_mode == kTabQ3 || p.tab_mode == kTabHybrid) && et < BN) build_threshold_row(sTab + et * kTabStride, n0 + et, g.N, p.e);
        RowCtx rc;
        if (A_PM1 && g.conv) rc = make_row(g, m0 + t);
        for (int i = 0; i < nkb; i++) {
            const int kb = kb0 + i;
            const int s = i % S;
            const uint32_t ph = (i / S) & 1;
            int kvalid = 128;
            if (A_PM1) {
                if (g.conv) {
                    kvalid = conv_kvalid(g, rc, kb_tap(g, kb));
                } else if (W_PM1) {
                    const int rem = g.K - kb * 128;
                    kvalid = rem < 128 ? rem : 128;
                }
            }
            mbar_wait(&plane_full[s], ph);
            if (i == 0 && threadIdx.x == 64) dbg_stamp(p, 1);
            mbar_wait(&op_empty[s], ph ^ 1);
            if ((i & 1) == grp) {
                a_job_any<A_PM1>(g.a_bits, sApl + (size_t)s * p.a_bytes, BM, t, tmem_lane + A_COL + s * 32, kvalid);
                tmem_wait_st();
            } else {
                uint8_t* bop = sBop + (size_t)s * BN * 128;
                const uint8_t* bpl = sBpl + (size_t)s * p.b_bytes;
                if (t < BN) b_job_any<W_PM1>(g.w_bits, bpl, BN, t, bop, 128);
                if (t + 128 < BN) b_job_any<W_PM1>(g.w_bits, bpl, BN, t + 128, bop, 128);
                fence_proxy_async_smem();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&plane_empty[s]);
                mbar_arrive(&op_full[s]);
            }
        }
        if (threadIdx.x == 64) dbg_stamp(p, 2);
        named_bar_sync(1, 256);  // threshold table complete (built before the mainloop)
        mbar_wait(accum_full, 0);
        tc_fence_after();
        if (threadIdx.x == 64) dbg_stamp(p, 3);
        const int m = m0 + t;
        constexpr int half = BN / 2;
        // int32 output: TMA stores from per-warp staging that reuses the (now idle)
        // pipeline buffers; packed output: direct stores (small problems only)
        const bool use_tma = p.out_mode == kOutTma && p.e.out_bits == 0 && m0 + q * 32 < g.M && !(kDev && p.exp_nostore);
        const bool use_lsu = p.out_mode == kOutLsu && p.e.out_bits == 0 && m0 + q * 32 < g.M && !(kDev && p.exp_nostore);
        uint8_t* stg = smem + (warp - 2) * kStgWarpBytes;
        uint32_t nst = 0;
#pragma unroll 1
        for (int c = grp * half; c < (grp + 1) * half; c += 32) {
            uint32_t acc[32];
            tmem_ld32(tmem_lane + c, acc);
            tmem_wait_ld();
            if (p.ksplit > 1) {  // partial sums -> this CTA's reduction buffer (reduced below)
                int32_t* red = reinterpret_cast<int32_t*>(smem);
#pragma unroll
                for (int j = 0; j < 8; j++)
                    *reinterpret_cast<uint4*>(red + split_red_index(t, c + 4 * j, BN)) =
                        make_uint4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
                continue;
            }
            if (kDev && p.exp_nostore) continue;
            if (use_tma) {
                uint8_t* b = stg + (nst & 1) * 4096;
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                stage_int32_chunk(acc, b, lane);
                fence_async_smem_cta();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmapY, smem_u32(b), n0 + c, m0 + q * 32);
                    bulk_commit();
                }
                nst++;
            } else if (use_lsu) {
                stage_int32_chunk(acc, stg, lane);
                __syncwarp();
                writeback_int32_block(stg, lane, reinterpret_cast<int32_t*>(p.Y), m0 + q * 32, g.M, n0 + c, g.N);
                __syncwarp();
            } else {
                epilogue_chunk(acc, m, n0 + c, c, g, p.e, p.Y, sTab, p.tab_mode);
            }
        }
        if (use_tma && lane == 0) bulk_wait<0>();
    }

    if (p.ksplit > 1) split_reduce_store<BN>(p, smem, m0, n0, sTab, warp, lane);
    tc_fence_before();
    __syncthreads();
    cta_stamp(p, 2);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, p.tmem_cols);
    }
    cta_stamp(p, 3);
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

// Packed operand [rows][RS][bits][Cw] (GEMM: RS = 1; conv weights: RS = R*S taps)
// viewed as a 4-D uint32 tensor {Cw, rows, bits, RS} (innermost first).  The box
// {4 words = 128 elements, box_rows, bits, 1} lands in shared memory as
// [plane][row][16 B] (conflict-free row-per-thread reads); coordinates
// {cb*4, row0, 0, tap}.
static bool make_plane_map(CUtensorMap* m, const uint32_t* base, int rows, int bits, int Cw, int RS, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)Cw, (cuuint64_t)rows, (cuuint64_t)bits, (cuuint64_t)RS};
    cuuint64_t strides[3] = {(cuuint64_t)RS * bits * Cw * 4, (cuuint64_t)Cw * 4, (cuuint64_t)bits * Cw * 4};
    cuuint32_t box[4] = {4, (cuuint32_t)box_rows, (cuuint32_t)bits, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Packed NHW[P][C] activations viewed as a 5-D uint32 tensor {Cw, W, bits, H, B};
// the box {4 words, bw * stride pixels (traversal stride = conv stride), bits, 1, 1}
// brings one output row's worth of input pixels for one filter tap and channel block,
// landing as [plane][pixel][16 B].  Out-of-frame coordinates are zero-filled.
static bool make_conv_act_map(CUtensorMap* m, const uint32_t* base, const Geom& g, int bw) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const cuuint64_t pix = (cuuint64_t)g.a_bits * g.Cw * 4;  // bytes per pixel record
    cuuint64_t dims[5] = {(cuuint64_t)g.Cw, (cuuint64_t)g.W, (cuuint64_t)g.a_bits, (cuuint64_t)g.H,
                          (cuuint64_t)(g.M / (g.Ho * g.Wo))};
    cuuint64_t strides[4] = {pix, (cuuint64_t)g.Cw * 4, pix * g.W, pix * g.W * g.H};
    cuuint32_t box[5] = {4, (cuuint32_t)(bw * g.stride), (cuuint32_t)g.a_bits, 1, 1};
    cuuint32_t estr[5] = {1, (cuuint32_t)g.stride, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<uint32_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// int32 output Y [M][N] as a 2-D tensor {N, M}; box {32 cols, 32 rows}, SWIZZLE_128B
// (the staging layout of stage_int32_chunk).  Needs N % 4 == 0 (16-byte row stride).
static bool make_out_map_i32(CUtensorMap* m, void* Y, int M, int N) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)N * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, Y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// packed output [M][bits][Nw] as a 3-D tensor {Nw, bits, M}; box {nwb, bits, 32}
static bool make_out_map_packed(CUtensorMap* m, void* Y, int M, int Nw, int bits, int nwb) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)Nw, (cuuint64_t)bits, (cuuint64_t)M};
    cuuint64_t strides[2] = {(cuuint64_t)Nw * 4, (cuuint64_t)bits * Nw * 4};
    cuuint32_t box[3] = {(cuuint32_t)nwb, (cuuint32_t)bits, 32};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, Y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C_in <= 128 (one channel block): the pixel record [bits][4 words] is contiguous, so
// the activations are viewed as a 4-D tensor {4*bits words, W, H, B} and one box row is
// a whole pixel (bits x 16 B): half (a2) to an eighth (a8) of the box rows of the
// plane-wise map, and the TMA unit's cost is per box row (scripts/tma_rate.cu).
static bool make_conv_act_map_merged(CUtensorMap* m, const uint32_t* base, const Geom& g, int bw) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const cuuint64_t pix = (cuuint64_t)g.a_bits * g.Cw * 4;
    cuuint64_t dims[4] = {(cuuint64_t)g.a_bits * g.Cw, (cuuint64_t)g.W, (cuuint64_t)g.H,
                          (cuuint64_t)(g.M / (g.Ho * g.Wo))};
    cuuint64_t strides[3] = {pix, pix * g.W, pix * g.W * g.H};
    cuuint32_t box[4] = {(cuuint32_t)(g.a_bits * g.Cw), (cuuint32_t)(bw * g.stride), 1, 1};
    cuuint32_t estr[4] = {1, (cuuint32_t)g.stride, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// prepared int8 W [N][Kp] bytes; box {128 bytes (one k-block), box_rows} with SWIZZLE_128B =
// the UMMA K-major SWIZZLE_128B operand layout of b_chunk_offset
static bool make_prep_i8_map(CUtensorMap* m, const uint8_t* base, int N, int Kp, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)Kp};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int stage_count(size_t per_stage, size_t fixed) {
    const size_t budget = 227 * 1024 - fixed;
    int S = (int)(budget / per_stage);
    return S > MAX_STAGES ? MAX_STAGES : S;
}

template <typename K>
static cudaError_t set_smem(K kfn) {
    return cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

template <int BNP, bool AP, bool WP>
static cudaError_t launch2(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, const Params& p,
                           int grid, size_t smem, cudaStream_t s) {
    auto kfn = p.acc_shift > 0 ? tc2_kernel<BNP, AP, WP, true> : tc2_kernel<BNP, AP, WP, false>;
    if constexpr (!AP) {  // fused residual instances (0/1 activations: the ResNet encodings)
        if (p.tab_mode == kTabResidual)
            kfn = p.acc_shift > 0 ? tc2_kernel<BNP, AP, WP, true, true> : tc2_kernel<BNP, AP, WP, false, true>;
    }
    cudaError_t e = set_smem(kfn);
    if (e != cudaSuccess) return e;
    kfn<<<grid, T2_THREADS, smem, s>>>(ta, tb, ty, p);
    return cudaGetLastError();
}

template <bool AP, bool WP>
static cudaError_t launch2_bn(int BNP, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty,
                              const Params& p, int grid, size_t smem, cudaStream_t s) {
    if (BNP == 256) return launch2<256, AP, WP>(ta, tb, ty, p, grid, smem, s);
    if (BNP == 128) return launch2<128, AP, WP>(ta, tb, ty, p, grid, smem, s);
    return launch2<64, AP, WP>(ta, tb, ty, p, grid, smem, s);
}

template <int BN, bool AP, bool WP>
static cudaError_t launch1(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, const Params& p,
                           dim3 grid, size_t smem, cudaStream_t s) {
    auto kfn = tc1_kernel<BN, AP, WP>;
    cudaError_t e = set_smem(kfn);
    if (e != cudaSuccess) return e;
    if (p.ksplit <= 1) {
        kfn<<<grid, T1_THREADS, smem, s>>>(ta, tb, ty, p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = dim3(T1_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = (unsigned)p.ksplit;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kfn, ta, tb, ty, p);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <bool AP, bool WP>
static cudaError_t launch1_bn(int BN, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty,
                              const Params& p, dim3 grid, size_t smem, cudaStream_t s) {
    if (BN == 256) return launch1<256, AP, WP>(ta, tb, ty, p, grid, smem, s);
    if (BN == 128) return launch1<128, AP, WP>(ta, tb, ty, p, grid, smem, s);
    return launch1<64, AP, WP>(ta, tb, ty, p, grid, smem, s);
}

}  // namespace tc

static int tc_kernel_override();

// The 2-CTA conv path fetches each output row's taps as one strided TMA box: the box is
// min(Wo, 128) pixels wide with element stride `stride`, so it needs width * stride <= 256
// (the box extent) and stride <= 8 (the largest TMA element stride).  Other convolutions run
// on the 1-CTA kernel, whose cp.async gathers take any stride.
static bool conv2_fits(const Geom& g) {
    const int bw = g.Wo <= 128 ? g.Wo : 128;
    return bw * g.stride <= 256 && g.stride <= 8;
}

// 2x2/2 max pooling fused into the 2-CTA kernel's epilogue (see pool_chunk)
bool tc_i8_pool_fusable(const Geom& g, const Epi& e) {
    return g.conv && e.pool == 2 && e.pool_stride == 2 && !e.pool_avg && e.out_bits > 0 && g.Ho % 2 == 0 &&
           g.Wo >= 2 && g.Wo <= 64 && g.M > 128 && conv2_fits(g) && tc_kernel_override() != 1;
}

namespace tc {
// apnn_prepare_weights_i8: packed W [N][w_bits][Kw] -> unscaled int8 operand rows [N][Kw*32]
// (u8 codes, or s8 +-1 with value-0 padding), 32 bytes per 32-element group in the
// recombination's element order (decode_01 / decode_pm1): the B tile of tc2_kernel as-is.
template <int NB, bool PM1>
__global__ void __launch_bounds__(256) prepare_i8_kernel(const uint32_t* __restrict__ W, int N, int K, int Kw,
                                                         uint8_t* __restrict__ out) {
    // x over a row's 32-element groups, y over rows, 32-bit index math (it also decodes the
    // activations of every both-prepared GEMM step: a flat 64-bit index division was its cost)
    for (int n = blockIdx.y * blockDim.y + threadIdx.y; n < N; n += gridDim.y * blockDim.y) {
        const uint32_t* wrow = W + (long long)n * NB * Kw;
        uint4* orow = reinterpret_cast<uint4*>(out + (long long)n * Kw * 32);
        for (int gidx = blockIdx.x * blockDim.x + threadIdx.x; gidx < Kw; gidx += gridDim.x * blockDim.x) {
            uint32_t pw[NB];
#pragma unroll
            for (int pl = 0; pl < NB; pl++) pw[pl] = __ldg(wrow + pl * Kw + gidx);
            uint32_t o[8];
            const int nv = K - gidx * 32;  // valid elements of this 32-element group
            const uint32_t vm = nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
            if (PM1) decode_pm1<true>(pw[0], vm, o);  // padding -> value 0
            else decode_01<NB>(pw, o);
            orow[gidx * 2] = make_uint4(o[0], o[1], o[2], o[3]);
            orow[gidx * 2 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
    }
}
}  // namespace tc

cudaError_t launch_prepare_weights_i8(const uint32_t* W, int N, int K, int w_bits, int enc, uint8_t* out, int sms,
                                      cudaStream_t s) {
    using namespace tc;
    const int Kw = (K + 127) / 128 * 4;
    if ((long long)N * Kw == 0) return cudaSuccess;
    dim3 threads(Kw >= 256 ? 256 : (Kw + 31) / 32 * 32, 1);
    threads.y = 256 / threads.x;
    dim3 gb((Kw + threads.x - 1) / threads.x, 1);
    const long long ry = ((long long)sms * 8 + gb.x - 1) / gb.x, need = ((long long)N + threads.y - 1) / threads.y;
    gb.y = (unsigned)(ry < need ? ry : need);
    if (gb.y > 65535) gb.y = 65535;
    const bool pm1 = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_PM1_A_01;
    if (pm1) { prepare_i8_kernel<1, true><<<gb, threads, 0, s>>>(W, N, K, Kw, out); }
    else {
        switch (w_bits) {
        case 1: prepare_i8_kernel<1, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        case 2: prepare_i8_kernel<2, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        case 3: prepare_i8_kernel<3, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        case 4: prepare_i8_kernel<4, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        case 5: prepare_i8_kernel<5, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        case 6: prepare_i8_kernel<6, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        case 7: prepare_i8_kernel<7, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        default: prepare_i8_kernel<8, false><<<gb, threads, 0, s>>>(W, N, K, Kw, out); break;
        }
    }
    count_launch();
    return cudaGetLastError();
}


bool tc_i8_supports(const Geom& g) {
    // GEMM and implicit-GEMM conv; K = 0 has no MMA to issue (handled by the popc variant)
    return g.K > 0 && g.M > 0 && g.N > 0;
}

static int nkb_dbg(const tc::Params& p) { return p.nkb; }

// experiment knob: APNN_TC_SCALED=0 disables the scaled operand form
static bool tc_scaled_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_TC_SCALED");
        v = s ? atoi(s) : 1;
    }
    return v != 0;
}

// epilogue store path.  Default (measured, 8192^3 w1a2, scripts/exp_time.py): int32
// output through TMA stores (441 us vs 481 coalesced-LSU vs 497 direct), packed
// output through coalesced LSU stores (equal to TMA, fewer constraints).
// Experiment knob APNN_EPI_STORE: 0 direct, 1 TMA, 2 coalesced LSU.
static int epi_store_mode(bool packed) {
    static int v = -2;
    if (v == -2) {
        const char* s = getenv("APNN_EPI_STORE");
        v = s ? atoi(s) : -1;
    }
    return v >= 0 ? v : (packed ? tc::kOutLsu : tc::kOutTma);
}

// merged pixel-record boxes for C_in <= 128 convs (experiment knob APNN_CONV_MERGE=0 disables)
constexpr int kMergedMaxBits = 4;  // [pixel][plane] rows of 16 B: up to 4-way LDS conflicts
static bool conv_merge_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_CONV_MERGE");
        v = s ? atoi(s) : 1;
    }
    return v != 0;
}

// largest split-K cluster (experiment knob APNN_SPLITZ).  Default 4: the paper's FC layer
// (M = 64, N = K = 1024, w1a2) measured 10.1 / 7.9 / 8.1 us at Z = 1 / 4 / 8.
static int split_zmax() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_SPLITZ");
        v = s ? atoi(s) : 4;
        if (v < 1) v = 1;
        if (v > 8) v = 8;
    }
    return v;
}

// variant knob for experiments: APNN_TC_KERNEL=1 forces the 1-CTA kernel
static int tc_kernel_override() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_TC_KERNEL");
        v = s ? atoi(s) : 0;
    }
    return v;
}

// 256-wide pair tiles as two N = 128 MMA halves (APNN_HALVES=1, read once; correct, slower)
static int halves_knob() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_HALVES");
        v = s ? atoi(s) : 0;
    }
    return v;
}

static cudaError_t launch_tc_i8_impl(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                                     int sms, cudaStream_t s, const uint8_t* Wprep, const TileCfg* force = nullptr) {
    using namespace tc;
    Params p;
    p.prep = Wprep ? 1 : 0;
    p.g = g;
    p.e = e;
    p.Y = Y;
    p.A = A;
    p.nkb = g.nchunks;
    p.tab_mode = kTabNone;
    if (e.res) {
        p.tab_mode = kTabResidual;  // v depends on the shortcut: no per-column thresholds
    } else if (e.out_bits > 0 && e.out_bits <= 2) {
        p.tab_mode = kTabQ3;
    } else if (e.out_bits > 2 && (unsigned long long)e.qmax * (unsigned long long)e.S <= 0xFFFFFFFFull) {
        p.tab_mode = kTabHybrid;  // 32-bit in-range division is exact (requant_hybrid)
    }
    p.out_mode = kOutDirect;
    p.nwb = 0;
    p.ksplit = 1;
    p.conv_merged = 0;
    p.pool_fused = e.pool ? 1 : 0;  // the ABI only forwards fusable pooling (tc_i8_pool_fusable)
    p.Hp = g.Ho / 2;
    p.Wp = g.Wo / 2;
    const int want_mode = epi_store_mode(e.out_bits > 0);
    p.acc_shift = 0;
    p.trace = nullptr;
    p.exp_nostore = 0;
    p.exp_nob = 0;
    p.halves = halves_knob();  // measured slower (8192^3 w1a2: 564 vs 455 us): N = 128 MMAs cost more
#if APNN_DEV
    p.exp_nostore = getenv("APNN_EXP_NOSTORE") ? 1 : 0;
    p.exp_nob = getenv("APNN_EXP_NOB") ? 1 : 0;
    const char* trace_path = getenv("APNN_TRACE");
    if (trace_path) {  // development only: allocates and synchronises (see the dump below)
        cudaMalloc(&p.trace, sizeof(unsigned long long) * (kTraceN * TR_N + 4 * kCtaTraceMax + 32));
        cudaMemset(p.trace, 0, sizeof(unsigned long long) * (kTraceN * TR_N + 4 * kCtaTraceMax + 32));
    }
#endif
    const int ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;
    bool two = (g.M > 128) && tc_kernel_override() != 1 && (!g.conv || conv2_fits(g));
    if (e.res && !two) return cudaErrorNotSupported;  // residual epilogue: 2-CTA kernel only (ABI checks first)
    if (Wprep && !two) return cudaErrorNotSupported;  // prepared W: 2-CTA kernel only
    // plain GEMMs (row f4): the tile -- CTA pair 256 x bn, or one CTA 128 x bn with a split-K
    // cluster of z CTAs -- comes from the paper's TLP/CI heuristic (tuner.cu), or the caller
    TileCfg cfg{0, 0, 0, 1, 0, 0.0};
    const bool tunable = !g.conv && !e.res && !Wprep && tc_kernel_override() == 0;
    if (force) {
        if (!tunable || !tile_cfg_valid(*force, g.M, g.N, g.K, e.out_bits > 0)) return cudaErrorNotSupported;
        cfg = *force;
    } else if (tunable) {
        cfg = tune_tiles(g.M, g.N, g.K, kTunerT, e.out_bits > 0);
    }
    if (cfg.kernel) two = cfg.kernel == 2;
    CUtensorMap ta, tb, ty;
    std::memset(&ty, 0, sizeof(ty));
    cudaError_t err;
    if (two) {
        const int BNP = cfg.kernel ? cfg.bn : (g.N > 128 ? 256 : (g.N > 64 ? 128 : 64));   // pair tile width
        const int brows = BNP / 2;
        p.b_bytes = p.prep ? 0u : 16u * brows * g.w_bits;
        p.conv_box_stride = 0;
        if (g.conv) {
            // row boxes per stage = output rows per CTA tile (conv_k below; even when pooling)
            const int bw = g.Wo <= 128 ? g.Wo : 128;
            const int nbox = g.Wo <= 128 ? (p.pool_fused ? (128 / g.Wo) & ~1 : 128 / g.Wo) : 1;
            p.conv_box_stride = (16 * bw * g.a_bits + 127) / 128 * 128;
            p.a_bytes = (uint32_t)(nbox * p.conv_box_stride);
            p.a_tx_bytes = (uint32_t)(nbox * 16 * bw * g.a_bits);
        } else {
            p.a_bytes = 16u * 128 * g.a_bits;
            p.a_tx_bytes = p.a_bytes;
        }
        {   // store staging per epilogue warp: int32 TMA 2 x 4 KB, int32 LSU 4 KB, packed one
            // {nwb, bits, 32} box; fused pooling uses 2 x 4 KB across the four warps
            const int nwb = BNP / 32 < 4 ? 4 : BNP / 32;
            int sw = 0;
            if (e.out_bits == 0) sw = want_mode == kOutTma ? 8192 : (want_mode == kOutLsu ? 4096 : 0);
            else if (want_mode != kOutDirect) sw = (e.out_bits * nwb * 128 + 1023) / 1024 * 1024;
            if (p.pool_fused && sw < 2048) sw = 2048;
            p.stg_warp = sw;
        }
        const size_t fixed = (size_t)256 * kTabStride * 4 + (2 * MAX_PSTAGES + 3 * MAX_STAGES + 6) * 8 +
                             T2_RECOMB_WARPS * 32 * 4 + 4 * (size_t)p.stg_warp + 1024;
        const size_t budget = 227 * 1024 - fixed;
        const size_t op_stage = (size_t)brows * 128, pl_stage = p.a_bytes + p.b_bytes;
        // Both ring depths must be EVEN: the two recombination teams take alternating
        // k-blocks, so with an even depth every stage (and its mbarrier phase sequence)
        // belongs to exactly one team.  With an odd depth a team can wait on a stage
        // whose barrier is two phases behind and try_wait.parity passes early (parity
        // aliasing).
        int S = 0, SP = 0;
        for (int s_try = MAX_STAGES; s_try >= 2; s_try -= 2) {  // deepest operand ring with >= s+2 plane stages
            if (budget < s_try * op_stage) continue;
            int sp = (int)((budget - s_try * op_stage) / pl_stage);
            if (sp > MAX_PSTAGES) sp = MAX_PSTAGES;
            sp &= ~1;
            if (sp >= s_try + 2 || (s_try == 2 && sp >= 2)) { S = s_try; SP = sp; break; }
        }
        if (S < 2) return cudaErrorInvalidConfiguration;
        p.stages = S;
        p.pstages = SP;
        {   // scaled operand form when the scaled accumulator cannot overflow int32
            const bool apm = g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_01_A_PM1;
            const bool wpm = g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_PM1_A_01;
            const int ka = apm ? 6 : 8 - g.a_bits, kw = wpm ? 6 : 8 - g.w_bits;
            const long long ma = apm ? 64 : (((1LL << g.a_bits) - 1) << ka);
            const long long mw = wpm ? 64 : (((1LL << g.w_bits) - 1) << kw);
            const bool safe = (long long)g.K * ma * mw < 2147483647LL;
            p.acc_shift = (safe && ka + kw > 0 && tc_scaled_enabled() && !p.prep) ? ka + kw : 0;  // prepared W is unscaled
        }
        p.tmem_cols = 512;
        int cta_tiles = (g.M + 127) / 128;
        p.conv_k = p.conv_bw = p.conv_segs = p.conv_nbox = 0;
        if (g.conv) {
            if (g.Wo <= 128) {
                p.conv_k = 128 / g.Wo;
                if (p.pool_fused) p.conv_k &= ~1;  // whole 2x2 grids per tile
                p.conv_bw = g.Wo;
                p.conv_nbox = p.conv_k;
                cta_tiles = (g.M / g.Wo + p.conv_k - 1) / p.conv_k;
            } else {
                p.conv_segs = (g.Wo + 127) / 128;
                p.conv_bw = 128;
                p.conv_nbox = 1;
                cta_tiles = (g.M / g.Wo) * p.conv_segs;
            }
            if (p.conv_bw * g.stride > 256 || g.stride > 8) return cudaErrorNotSupported;  // conv2_fits said so
        }
        p.tiles_m = (cta_tiles + 1) / 2;
        // tiles cover [0, N); the packed path also writes the N padding words (zero)
        const int tiles_n = (g.N + BNP - 1) / BNP;
        p.num_tiles = p.tiles_m * tiles_n;
        int clusters = sms / 2;
        if (clusters > p.num_tiles) clusters = p.num_tiles;
        const size_t smem = (size_t)S * op_stage + (size_t)SP * pl_stage + fixed - 1024 + 64;
        if (g.conv) {
            p.conv_merged = (g.CB == 1 && g.a_bits <= kMergedMaxBits && conv_merge_enabled()) ? 1 : 0;
            if (p.conv_merged ? !make_conv_act_map_merged(&ta, A, g, p.conv_bw)
                              : !make_conv_act_map(&ta, A, g, p.conv_bw))
                return cudaErrorInvalidValue;
        } else if (!make_plane_map(&ta, A, g.M, g.a_bits, g.Cw, 1, 128)) {
            return cudaErrorInvalidValue;
        }
        if (p.prep) {
            // GEMM: [N][Kp]; conv: [C_out][R*S*Cp] (taps x channel blocks) -- k-block kb at byte kb*128
            if (!make_prep_i8_map(&tb, Wprep, g.N, g.RS * g.Cw * 32, brows)) return cudaErrorInvalidValue;
        } else if (!make_plane_map(&tb, W, g.N, g.w_bits, g.Cw, g.RS, brows)) {
            return cudaErrorInvalidValue;
        }
        p.nwb = BNP / 32 < 4 ? 4 : BNP / 32;
        if (want_mode == kOutLsu) {
            p.out_mode = (e.out_bits > 0 || g.N % 4 == 0) ? kOutLsu : kOutDirect;
        } else if (want_mode == kOutTma) {
            if (e.out_bits == 0) {
                p.out_mode = (g.N % 4 == 0 && make_out_map_i32(&ty, Y, g.M, g.N)) ? kOutTma : kOutDirect;
            } else {
                const int Nw = (g.N + 127) / 128 * 4;
                p.out_mode = make_out_map_packed(&ty, Y, g.M, Nw, e.out_bits, p.nwb) ? kOutTma : kOutDirect;
            }
        }
        switch (g.enc) {
        case APNN_ENC_01_01: err = launch2_bn<false, false>(BNP, ta, tb, ty, p, clusters * 2, smem, s); break;
        case APNN_ENC_PM1_PM1: err = launch2_bn<true, true>(BNP, ta, tb, ty, p, clusters * 2, smem, s); break;
        case APNN_ENC_W_PM1_A_01: err = launch2_bn<false, true>(BNP, ta, tb, ty, p, clusters * 2, smem, s); break;
        default: err = launch2_bn<true, false>(BNP, ta, tb, ty, p, clusters * 2, smem, s); break;
        }
    } else {
        int BN = g.N > 128 ? 256 : (g.N > 64 ? 128 : 64);
        // split-K over a cluster of Z CTAs when the output tiles alone leave SMs idle
        p.ksplit = 1;
        if (cfg.kernel) {
            BN = cfg.bn;
            p.ksplit = cfg.z;
        } else if (tc_kernel_override() != 3) {
            const int BNs = g.N > 1024 ? 128 : 64;
            const long long tiles = (long long)((g.M + BM - 1) / BM) * ((ncols + BNs - 1) / BNs);
            int Z = 1;
            const int zmax = split_zmax();
            while (Z < zmax && 2 * Z <= g.nchunks && tiles * 2 * Z <= sms) Z *= 2;
            if (Z > 1) {
                p.ksplit = Z;
                BN = BNs;
            }
        }
        p.a_bytes = 16u * BM * g.a_bits;
        p.b_bytes = 16u * BN * g.w_bits;
        const size_t fixed = (size_t)BN * kTabStride * 4 + (4 * MAX_STAGES + 4) * 8 + 1024;
        int S = stage_count((size_t)BN * 128 + p.a_bytes + p.b_bytes, fixed);
        if (S < 2) return cudaErrorInvalidConfiguration;
        if (p.ksplit > 1) {
            // a split CTA runs only ~nkb/Z k-blocks: a shallow ring keeps TMEM (BN + 32 S
            // columns) and shared memory small, so co-resident CTAs never wait on tcgen05.alloc
            const int per = (g.nchunks + p.ksplit - 1) / p.ksplit;
            const size_t stage = (size_t)BN * 128 + p.a_bytes + p.b_bytes, red = (size_t)BM * BN * 4;
            const int fit = (int)((227 * 1024 - fixed - red) / stage);
            S = per < 2 ? 2 : (per < S ? per : S);
            if (S > fit) S = fit;
            if (S < 2) return cudaErrorInvalidConfiguration;
        }
        p.stages = S;
        p.pstages = S;
        uint32_t cols = BN + 32 * S, pow2 = 32;
        while (pow2 < cols) pow2 <<= 1;
        p.tmem_cols = pow2;
        p.tiles_m = 0;
        p.num_tiles = 0;
        const size_t smem = (size_t)S * ((size_t)BN * 128 + p.a_bytes + p.b_bytes) + fixed - 1024 + 64 +
                            (p.ksplit > 1 ? (size_t)BM * BN * 4 : 0);
        if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
        if (!make_plane_map(&ta, A, g.conv ? 1 : g.M, g.a_bits, g.Cw, 1, BM)) return cudaErrorInvalidValue;
        if (!make_plane_map(&tb, W, g.N, g.w_bits, g.Cw, g.RS, BN)) return cudaErrorInvalidValue;
        dim3 grid((g.M + BM - 1) / BM, (ncols + BN - 1) / BN, p.ksplit);
        // int32 output through TMA stores, staged in the idle pipeline buffers (8 warps x 8 KB)
        if (e.out_bits == 0 && g.N % 4 == 0 && want_mode != kOutDirect &&
            (size_t)S * ((size_t)BN * 128 + p.a_bytes + p.b_bytes) >= 8 * kStgWarpBytes) {
            if (want_mode == kOutLsu) p.out_mode = kOutLsu;
            else p.out_mode = make_out_map_i32(&ty, Y, g.M, g.N) ? kOutTma : kOutDirect;
        }
        switch (g.enc) {
        case APNN_ENC_01_01: err = launch1_bn<false, false>(BN, ta, tb, ty, p, grid, smem, s); break;
        case APNN_ENC_PM1_PM1: err = launch1_bn<true, true>(BN, ta, tb, ty, p, grid, smem, s); break;
        case APNN_ENC_W_PM1_A_01: err = launch1_bn<false, true>(BN, ta, tb, ty, p, grid, smem, s); break;
        default: err = launch1_bn<true, false>(BN, ta, tb, ty, p, grid, smem, s); break;
        }
    }
#if APNN_DEV
    if (p.trace) {  // development only: synchronous dump
        static unsigned long long host[kTraceN * TR_N + 4 * kCtaTraceMax + 32];
        cudaStreamSynchronize(s);
        cudaMemcpy(host, p.trace, sizeof(host), cudaMemcpyDeviceToHost);
        cudaFree(p.trace);
        if (FILE* f = fopen(trace_path, "wb")) {
            int hdr[4] = {kTraceN, TR_N, nkb_dbg(p), p.stages};
            fwrite(hdr, sizeof(hdr), 1, f);
            fwrite(host, sizeof(host), 1, f);
            fclose(f);
        }
    }
#endif
    count_launch();
    return err;
}

cudaError_t launch_tc_i8(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y, int sms,
                         cudaStream_t s) {
    return launch_tc_i8_impl(A, W, g, e, Y, sms, s, nullptr);
}

cudaError_t launch_tc_i8_tiled(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                               const TileCfg& cfg, int sms, cudaStream_t s) {
    return launch_tc_i8_impl(A, W, g, e, Y, sms, s, nullptr, &cfg);
}

cudaError_t launch_tc_i8_prepared(const uint32_t* A, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                  int sms, cudaStream_t s) {
    return launch_tc_i8_impl(A, nullptr, g, e, Y, sms, s, Wp);
}

}  // namespace apnn
