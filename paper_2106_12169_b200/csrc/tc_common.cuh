// tc_common.cuh -- building blocks of the tcgen05 kind::i8 kernels (gemm_tc.cu):
//   * plane -> int8 recombination jobs (the operand-side bit combination),
//   * the epilogue: int32 store, or the fused element-wise routine
//     (requantise -> bit-decompose -> pack along N).
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace apnn {
namespace tc {

// Element order inside a 32-element group (identical for A and B, so the dot
// product is unchanged): output word j (j = 0..7) holds elements j, j+8, j+16,
// j+24 in its bytes 0..3.  Word j of group gi sits at K-byte 32*gi + 4*j.

__device__ __forceinline__ uint32_t sel4(const uint4& v, int gi) {
    return gi == 0 ? v.x : gi == 1 ? v.y : gi == 2 ? v.z : v.w;
}

// 0/1 codes with NB planes -> u8 lanes: byte = sum_t bit_t << t  (Eq. bitCombination
// applied to the operand: one shift + one masked OR per plane and word)
template <int NB>
__device__ __forceinline__ void decode_01(const uint32_t (&pw)[NB], uint32_t (&out)[8]) {
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

// +-1 plane -> s8 lanes: bit 1 -> +1 (0x01), bit 0 -> -1 (0xFF);
// elements outside `vm` decode to 0 (padded K of Case II).
template <bool kMasked>
__device__ __forceinline__ void decode_pm1(uint32_t pw, uint32_t vm, uint32_t (&out)[8]) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint32_t s = (pw >> j) & 0x01010101u;
        uint32_t o = s * 0xFFFFFF02u + 0xFFFFFFFFu;  // 0xFF - 0xFE*s per byte, no borrows
        if (kMasked) o &= ((vm >> j) & 0x01010101u) * 0xFFu;
        out[j] = o;
    }
}

__device__ __forceinline__ uint32_t valid_mask(int kvalid, int gi) {
    const int nv = kvalid - gi * 32;
    return nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
}

// ---- scaled decodes (FMA-pipe form).  The operand bytes are the codes times a
// power of two: 0/1 codes with NB planes are top-aligned (x 2^(8-NB)), +-1 values
// are +-64.  The int32 result is then Y * 2^(kA+kB), shifted back exactly in the
// epilogue (the host only picks this form when K*max|a'|*max|w'| < 2^31).  Each
// plane-word costs one LOP3 mask (ALU) + one IMAD shift-and-add (FMA pipe) instead
// of SHF + LOP3 on the ALU; the multipliers live in constant memory so ptxas keeps
// real IMADs instead of strength-reducing them back to ALU shifts.
__constant__ uint32_t kPow2[16] = {1u, 2u, 4u, 8u, 16u, 32u, 64u, 128u, 256u, 512u, 1024u, 2048u, 4096u,
                                   8192u, 16384u, 32768u};
__constant__ uint32_t kPm1Mul[8] = {0xFFFFFF80u, 0xFFFFFFC0u, 0xFFFFFFE0u, 0xFFFFFFF0u,
                                    0xFFFFFFF8u, 0xFFFFFFFCu, 0xFFFFFFFEu, 0xFFFFFFFFu};  // -(128 >> j)

template <int NB>
__device__ __forceinline__ void decode_01_scaled(const uint32_t (&pw)[NB], uint32_t (&out)[8]) {
    constexpr int k = 8 - NB;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        uint32_t o = 0;
#pragma unroll
        for (int t = 0; t < NB; t++) {
            const int sh = k + t - j;
            const uint32_t x = pw[t] & (0x01010101u << j);
            if (sh >= 0) o = x * kPow2[sh] + o;   // disjoint bits: add == or
            else o |= x >> (-sh);
        }
        out[j] = o;
    }
}
// +-1 -> +-64: byte = 192 - 128*bit (no borrows); masked elements -> 0
template <bool kMasked>
__device__ __forceinline__ void decode_pm1_scaled(uint32_t pw, uint32_t vm, uint32_t (&out)[8]) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint32_t x = pw & (0x01010101u << j);
        uint32_t o = x * kPm1Mul[j] + 0xC0C0C0C0u;
        if (kMasked) o &= ((vm >> j) & 0x01010101u) * 0xFFu;
        out[j] = o;
    }
}

template <int NB, bool PM1, bool SCALED = false>
__device__ __forceinline__ void decode_group(const uint4 (&v)[NB], int gi, int kvalid, uint32_t (&o)[8]) {
    uint32_t pw[NB];
#pragma unroll
    for (int pl = 0; pl < NB; pl++) pw[pl] = sel4(v[pl], gi);
    if (PM1) {
        if (SCALED) {
            if (kvalid >= 128) decode_pm1_scaled<false>(pw[0], 0u, o);
            else decode_pm1_scaled<true>(pw[0], valid_mask(kvalid, gi), o);
        } else {
            if (kvalid >= 128) decode_pm1<false>(pw[0], 0u, o);
            else decode_pm1<true>(pw[0], valid_mask(kvalid, gi), o);
        }
    } else {
        if (SCALED) decode_01_scaled<NB>(pw, o);
        else decode_01<NB>(pw, o);
    }
}

// A job: one 128-element k-block of one A row -> 32 TMEM columns of the thread's lane.
// planes: smem [plane][rows][16 B] as written by the TMA box.
template <int NB, bool PM1>
__device__ __forceinline__ void a_job(const uint8_t* planes, int rows, int row, uint32_t taddr, int kvalid) {
    const uint4* src = reinterpret_cast<const uint4*>(planes);
    uint4 v[NB];
#pragma unroll
    for (int pl = 0; pl < NB; pl++) v[pl] = src[pl * rows + row];
#pragma unroll
    for (int gi = 0; gi < 4; gi++) {
        uint32_t o[8];
        decode_group<NB, PM1>(v, gi, kvalid, o);
        sm100::tmem_st8(taddr + gi * 8, o);
    }
}

// B operand tile layout in shared memory (one 128-byte K row per N row):
//   APNN_B_SWIZZLE128 (default): UMMA K-major SWIZZLE_128B atoms of 8 rows x 128 B,
//     row r, 16-byte chunk c at (r>>3)*1024 + (r&7)*128 + ((c ^ (r&7))*16)
//   otherwise: K-major no-swizzle core matrices, chunk c at (r>>3)*1024 + c*128 + (r&7)*16.
// Both are conflict-free for the row-per-thread 16-byte stores.
#ifndef APNN_B_SWIZZLE128
#define APNN_B_SWIZZLE128 1
#endif
__device__ __forceinline__ uint32_t b_chunk_offset(int row, int c) {
#if APNN_B_SWIZZLE128
    return (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4);
#else
    return (row >> 3) * 1024 + c * 128 + (row & 7) * 16;
#endif
}
// descriptor increment (16-byte units) between consecutive 32-byte K steps
#if APNN_B_SWIZZLE128
constexpr uint32_t kBDescKStep = 2;
#else
constexpr uint32_t kBDescKStep = 16;
#endif
// smem descriptor of k-step kk (32 bytes of K) of a B tile starting at `base` (1024-aligned)
__device__ __forceinline__ uint64_t b_desc(uint32_t base, int kk) {
#if APNN_B_SWIZZLE128
    return sm100::umma_desc_sw128(base + kk * 32, 1024);
#else
    return sm100::umma_desc_noswizzle(base + kk * 256, 128, 1024);
#endif
}

// B job: one 128-element k-block of one B row -> the B operand tile layout above.
template <int NB, bool PM1>
__device__ __forceinline__ void b_job(const uint8_t* planes, int rows, int row, uint8_t* bop, int kvalid) {
    const uint4* src = reinterpret_cast<const uint4*>(planes);
    uint4 v[NB];
#pragma unroll
    for (int pl = 0; pl < NB; pl++) v[pl] = src[pl * rows + row];
#pragma unroll
    for (int gi = 0; gi < 4; gi++) {
        uint32_t o[8];
        decode_group<NB, PM1>(v, gi, kvalid, o);
        *reinterpret_cast<uint4*>(bop + b_chunk_offset(row, 2 * gi)) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(bop + b_chunk_offset(row, 2 * gi + 1)) = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

// Recombination step with early release of the plane stage: load this thread's
// planes and decode them into the 32 int8-lane words in registers (this consumes
// the shared-memory loads, so the release below cannot overtake them -- releasing
// right after issuing the LDS raced with the TMA refill: whole rows read the next
// use of the stage), release the plane stage (the TMA can refill it), then wait
// for the operand stage to be free and store.
// Plane pl of row `row` is the 16-byte chunk src[pl * pstride + row * rstride] of the
// stage: [plane][row][16 B] (pstride = rows, rstride = 1; GEMM and the W operand) or
// [row][plane][16 B] (pstride = 1, rstride = NB; conv rows fetched as whole pixel records).
template <int NB, bool PM1, bool IS_A, bool SCALED>
__device__ __forceinline__ void recomb_step(const uint8_t* planes, int pstride, int rstride, int row,
                                            uint64_t* plane_empty, uint64_t* op_empty, uint32_t op_parity,
                                            uint32_t taddr, uint8_t* bop, int kvalid, int lane,
                                            volatile uint32_t* dep_slot) {
    const uint4* src = reinterpret_cast<const uint4*>(planes);
    uint4 v[NB];
#pragma unroll
    for (int pl = 0; pl < NB; pl++) v[pl] = src[pl * pstride + row * rstride];
    // The release below must not overtake the plane loads: neither mbarrier.arrive's
    // release semantics nor program order make the hardware wait for in-flight LDS.
    // A store of a value that depends on one register of every LDS.128 forces all of
    // them to complete first.  (Without it the TMA refill of this plane stage raced
    // the tail of the LDS: the k-block one ring depth later leaked into whole rows,
    // ~20 tiles per 8192^3 run -- scripts/race_check.py.)
    uint32_t dep = 0;
#pragma unroll
    for (int pl = 0; pl < NB; pl++) dep ^= v[pl].x;
    *dep_slot = dep;
    uint32_t o[4][8];
#pragma unroll
    for (int gi = 0; gi < 4; gi++) decode_group<NB, PM1, SCALED>(v, gi, kvalid, o[gi]);
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(plane_empty);
    sm100::mbar_wait(op_empty, op_parity);
    if (IS_A) {
#pragma unroll
        for (int gi = 0; gi < 4; gi++) sm100::tmem_st8(taddr + gi * 8, o[gi]);
    } else {
#pragma unroll
        for (int gi = 0; gi < 4; gi++) {
            *reinterpret_cast<uint4*>(bop + b_chunk_offset(row, 2 * gi)) =
                make_uint4(o[gi][0], o[gi][1], o[gi][2], o[gi][3]);
            *reinterpret_cast<uint4*>(bop + b_chunk_offset(row, 2 * gi + 1)) =
                make_uint4(o[gi][4], o[gi][5], o[gi][6], o[gi][7]);
        }
    }
}

template <bool PM1, bool IS_A, bool SCALED>
__device__ __forceinline__ void recomb_step_any(int nb, const uint8_t* planes, int pstride, int rstride, int row,
                                                uint64_t* plane_empty, uint64_t* op_empty, uint32_t op_parity,
                                                uint32_t taddr, uint8_t* bop, int kvalid, int lane,
                                                volatile uint32_t* dep_slot) {
#define APNN_RS(N_) recomb_step<N_, PM1, IS_A, SCALED>(planes, pstride, rstride, row, plane_empty, op_empty, op_parity, taddr, bop, kvalid, lane, dep_slot)
    if (PM1) { recomb_step<1, true, IS_A, SCALED>(planes, pstride, rstride, row, plane_empty, op_empty, op_parity, taddr, bop, kvalid, lane, dep_slot); return; }
    switch (nb) {  // warp-uniform
    case 1: APNN_RS(1); break;
    case 2: APNN_RS(2); break;
    case 3: APNN_RS(3); break;
    case 4: APNN_RS(4); break;
    case 5: APNN_RS(5); break;
    case 6: APNN_RS(6); break;
    case 7: APNN_RS(7); break;
    default: APNN_RS(8); break;
    }
#undef APNN_RS
}

template <bool PM1>
__device__ __forceinline__ void a_job_any(int nb, const uint8_t* planes, int rows, int row, uint32_t taddr,
                                          int kvalid) {
    if (PM1) { a_job<1, true>(planes, rows, row, taddr, kvalid); return; }
    switch (nb) {  // warp-uniform
    case 1: a_job<1, false>(planes, rows, row, taddr, kvalid); break;
    case 2: a_job<2, false>(planes, rows, row, taddr, kvalid); break;
    case 3: a_job<3, false>(planes, rows, row, taddr, kvalid); break;
    case 4: a_job<4, false>(planes, rows, row, taddr, kvalid); break;
    case 5: a_job<5, false>(planes, rows, row, taddr, kvalid); break;
    case 6: a_job<6, false>(planes, rows, row, taddr, kvalid); break;
    case 7: a_job<7, false>(planes, rows, row, taddr, kvalid); break;
    default: a_job<8, false>(planes, rows, row, taddr, kvalid); break;
    }
}

template <bool PM1>
__device__ __forceinline__ void b_job_any(int nb, const uint8_t* planes, int rows, int row, uint8_t* bop,
                                          int kvalid) {
    if (PM1) { b_job<1, true>(planes, rows, row, bop, kvalid); return; }
    switch (nb) {
    case 1: b_job<1, false>(planes, rows, row, bop, kvalid); break;
    case 2: b_job<2, false>(planes, rows, row, bop, kvalid); break;
    case 3: b_job<3, false>(planes, rows, row, bop, kvalid); break;
    case 4: b_job<4, false>(planes, rows, row, bop, kvalid); break;
    case 5: b_job<5, false>(planes, rows, row, bop, kvalid); break;
    case 6: b_job<6, false>(planes, rows, row, bop, kvalid); break;
    case 7: b_job<7, false>(planes, rows, row, bop, kvalid); break;
    default: b_job<8, false>(planes, rows, row, bop, kvalid); break;
    }
}

// ------------------------------------------------------- conv A-row gather
// Implicit GEMM (APConv as GEMM): k-block kb is filter tap
// rs = kb / CB and channel block cb = kb % CB; A row m is output pixel
// (b, ho, wo) and reads input pixel (ho*st + r - pad, wo*st + s - pad).
struct KbTap {
    int r, s, cb;
};
__device__ __forceinline__ KbTap kb_tap(const Geom& g, int kb) {
    KbTap t;
    const int rs = kb / g.CB;
    t.cb = kb - rs * g.CB;
    t.r = rs / g.S;
    t.s = rs - t.r * g.S;
    return t;
}
// plane-0 address of the chunk, or nullptr when the tap is out of frame / row >= M
__device__ __forceinline__ const uint32_t* conv_a_src(const uint32_t* X, const Geom& g, const RowCtx& c,
                                                      const KbTap& t) {
    const int hi = c.hb + t.r, wi = c.wb + t.s;
    if (!c.valid || hi < 0 || hi >= g.H || wi < 0 || wi >= g.W) return nullptr;
    return X + ((c.pix + (long long)hi * g.W + wi) * g.a_bits) * g.Cw + t.cb * 4;
}
// logical elements of the chunk for +-1 activations: 0 out of frame (value-domain
// zero padding), else the unpadded channels of block cb
__device__ __forceinline__ int conv_kvalid(const Geom& g, const RowCtx& c, const KbTap& t) {
    const int hi = c.hb + t.r, wi = c.wb + t.s;
    if (!c.valid || hi < 0 || hi >= g.H || wi < 0 || wi >= g.W) return 0;
    const int rem = g.C - t.cb * 128;
    return rem < 128 ? rem : 128;
}
// one warp gathers `rows` A rows (lane, lane+32, ...) of k-block kb into the
// plane stage [plane][rows][16 B] with zero-filling cp.async, then arms the
// stage's mbarrier (one .noinc arrival per lane).
template <int kRowsPerLane>
__device__ __forceinline__ void conv_gather_kb(const uint32_t* X, const Geom& g, const RowCtx (&rc)[kRowsPerLane],
                                               int kb, uint8_t* stage, int rows, int lane, uint64_t* bar) {
    const KbTap t = kb_tap(g, kb);
    const uint32_t sbase = sm100::smem_u32(stage);
#pragma unroll
    for (int i = 0; i < kRowsPerLane; i++) {
        const int row = lane + 32 * i;
        if (row >= rows) break;
        const uint32_t* src = conv_a_src(X, g, rc[i], t);
        for (int pl = 0; pl < g.a_bits; pl++)
            sm100::cp_async16_zfill(sbase + (pl * rows + row) * 16, src ? src + (long long)pl * g.Cw : X,
                                    src ? 16u : 0u);
    }
    sm100::cp_async_mbar_arrive_noinc(bar);
}

// ------------------------------------------------------------------ epilogue
// Per-column requantisation table (built once per output tile in shared memory).
// For column n, with y' = -y if alpha < 0 else y (|y| <= 2^31 - 1 by the host
// overflow check, so y' never overflows), q = clamp(floor((alpha y + beta)/S), 0, Q)
// is a non-decreasing function of y', and
//   q >= k  <=>  y' > U_k,   U_k = ceil((kS - beta)/alpha) - 1   (alpha > 0)
//                                = -floor((kS - beta)/alpha) - 1  (alpha < 0)
//                                = INT32_MIN if beta >= kS else INT32_MAX (alpha = 0)
// (clamped to int32: exact for int32 y').  Row layout, kTabStride int32:
//   [0] sign  [1] U_1  [2] U_2  [3] U_3  [4] U_Q  [5] alpha  [6] beta  [7] unused
// Padding columns (n >= N) get all thresholds INT32_MAX and alpha = beta = 0: q = 0.
constexpr int kTabStride = 8;
enum { kTabNone = 0, kTabQ3 = 1, kTabHybrid = 2, kTabResidual = 3 };

__device__ __forceinline__ long long floor_div64(long long a, long long b) {
    long long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

__device__ __forceinline__ int32_t threshold_k(long long al, long long be, long long S, int k) {
    const long long num = (long long)k * S - be;
    long long U;
    if (al > 0) U = -floor_div64(-num, al) - 1;  // ceil(num/al) - 1
    else if (al < 0) U = -floor_div64(num, al) - 1;
    else U = (be >= (long long)k * S) ? (long long)INT32_MIN : 0x7FFFFFFFLL;
    if (U < INT32_MIN) U = INT32_MIN;
    if (U > 0x7FFFFFFFLL) U = 0x7FFFFFFFLL;
    return (int32_t)U;
}

__device__ __forceinline__ void build_threshold_row(int32_t* row, int n, int N, const Epi& e) {
    const int Q = e.qmax;
    if (n >= N) {
        *reinterpret_cast<int4*>(row) = make_int4(1, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF);
        *reinterpret_cast<int4*>(row + 4) = make_int4(0x7FFFFFFF, 0, 0, 0);
        return;
    }
    const long long al = epi_alpha(e, n), be = epi_beta(e, n), S = e.S;
    int32_t u[3];
#pragma unroll
    for (int k = 1; k <= 3; k++) u[k - 1] = (k <= Q) ? threshold_k(al, be, S, k) : 0x7FFFFFFF;
    *reinterpret_cast<int4*>(row) = make_int4(al < 0 ? -1 : 1, u[0], u[1], u[2]);
    *reinterpret_cast<int4*>(row + 4) = make_int4(threshold_k(al, be, S, Q), (int32_t)al, (int32_t)be, 0);
}

// Q <= 3 (out_bits <= 2): with c_k = [y' > U_k] monotone (c1 >= c2 >= c3),
// q = c1 + c2 + c3, so bit 1 of q is c2 and bit 0 is c1 ^ c2 ^ c3.  Plane words
// are assembled straight from the comparisons (no byte staging).
__device__ __forceinline__ void requant_chunk_words_q3(const uint32_t (&acc)[32], const int32_t* tab, int lc,
                                                       uint32_t& w0, uint32_t& w1) {
    w0 = 0;
    w1 = 0;
#pragma unroll
    for (int i = 0; i < 32; i++) {
        const int4 h = *reinterpret_cast<const int4*>(tab + (lc + i) * kTabStride);
        const int32_t yp = (int32_t)acc[i] * h.x;
        const bool c1 = yp > h.y, c2 = yp > h.z, c3 = yp > h.w;
        if (c1 ^ c2 ^ c3) w0 |= 1u << i;
        if (c2) w1 |= 1u << i;
    }
}

// Q >= 7 (out_bits >= 3), host-checked Q*S < 2^32: the two clamps come from the
// table; in between S <= v < Q*S, so v = alpha*y + beta is exact in 32-bit
// (wrap-around) arithmetic and q = v / S is a 32-bit division by the layer
// constant: an fp32 estimate (off by at most one) and one exact correction.
__device__ __forceinline__ uint32_t requant_hybrid(const int32_t* row, int32_t y, uint32_t S, float invS,
                                                   uint32_t Q) {
    const int4 h = *reinterpret_cast<const int4*>(row);
    const int4 h2 = *reinterpret_cast<const int4*>(row + 4);
    const int32_t yp = y * h.x;
    const uint32_t v = (uint32_t)h2.y * (uint32_t)y + (uint32_t)h2.z;
    uint32_t q = __float2uint_rz(__uint2float_rn(v) * invS);
    const int32_t r = (int32_t)(v - q * S);
    q = r < 0 ? q - 1 : (r >= (int32_t)S ? q + 1 : q);
    q = yp > h2.x ? Q : q;
    return yp > h.y ? q : 0u;
}

// 32 accumulators -> 32 codes as bytes (byte i of qb[j] = q of column nb + 4j + i)
__device__ __forceinline__ void requant_chunk_bytes(const uint32_t (&acc)[32], int nb, int lc, const Geom& g,
                                                    const Epi& e, const int32_t* tab, int tab_mode,
                                                    uint32_t (&qb)[8]) {
#pragma unroll
    for (int i = 0; i < 8; i++) qb[i] = 0;
    if (tab_mode == kTabQ3) {
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int4 h = *reinterpret_cast<const int4*>(tab + (lc + i) * kTabStride);
            const int32_t yp = (int32_t)acc[i] * h.x;
            const uint32_t q = (uint32_t)(yp > h.y) + (uint32_t)(yp > h.z) + (uint32_t)(yp > h.w);
            qb[i >> 2] |= q << (8 * (i & 3));
        }
    } else if (tab_mode == kTabHybrid) {
        const uint32_t S = (uint32_t)e.S, Q = (uint32_t)e.qmax;
#pragma unroll
        for (int i = 0; i < 32; i++)
            qb[i >> 2] |= requant_hybrid(tab + (lc + i) * kTabStride, (int32_t)acc[i], S, e.invS, Q) << (8 * (i & 3));
    } else {
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int n = nb + i;
            uint32_t qv = 0;
            if (n < g.N) qv = requant(e, (int32_t)acc[i], epi_alpha(e, n), epi_beta(e, n));
            qb[i >> 2] |= qv << (8 * (i & 3));
        }
    }
}

// 32 byte codes (byte i of qb[j] = code 4j + i) -> 8 plane words (bit i of words[t] = bit t of
// code i): the 32 x 8 bit matrix is four 8 x 8 blocks, each transposed with three delta swaps
// (bit 8r + c <-> 8c + r), then byte permutes gather plane t's byte from the four blocks --
// ~100 ops for all 8 planes instead of ~48 per plane (checked against the per-bit definition)
__device__ __forceinline__ void bytes_to_words_t(const uint32_t (&qb)[8], uint32_t (&words)[8]) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int b = 0; b < 4; b++) {
        uint32_t x = qb[2 * b], y = qb[2 * b + 1], t;
        t = (x ^ (x >> 7)) & 0x00AA00AAu;  x = x ^ t ^ (t << 7);
        t = (y ^ (y >> 7)) & 0x00AA00AAu;  y = y ^ t ^ (t << 7);
        t = (x ^ (x >> 14)) & 0x0000CCCCu; x = x ^ t ^ (t << 14);
        t = (y ^ (y >> 14)) & 0x0000CCCCu; y = y ^ t ^ (t << 14);
        t = (x ^ (y << 4)) & 0xF0F0F0F0u;  x ^= t; y ^= t >> 4;
        lo[b] = x;
        hi[b] = y;
    }
#pragma unroll
    for (int t = 0; t < 8; t++) {
        const uint32_t* L = t < 4 ? lo : hi;
        const uint32_t sel = (uint32_t)(t & 3) | ((uint32_t)((t & 3) + 4) << 4);
        words[t] = __byte_perm(__byte_perm(L[0], L[1], sel), __byte_perm(L[2], L[3], sel), 0x5410);
    }
}

// The inverse: 8 plane words -> 32 byte codes (byte i of qb[j] = code 4j + i).  The 8 x 8 block
// transpose is an involution, so the byte permutes run first and the delta swaps second.
__device__ __forceinline__ void words_to_bytes_t(const uint32_t (&words)[8], uint32_t (&qb)[8]) {
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const uint32_t sel = (uint32_t)b | ((uint32_t)(b + 4) << 4);  // byte b of two words -> bytes 0, 1
        uint32_t x = __byte_perm(__byte_perm(words[0], words[1], sel), __byte_perm(words[2], words[3], sel), 0x5410);
        uint32_t y = __byte_perm(__byte_perm(words[4], words[5], sel), __byte_perm(words[6], words[7], sel), 0x5410);
        uint32_t t;
        t = (x ^ (x >> 7)) & 0x00AA00AAu;  x = x ^ t ^ (t << 7);
        t = (y ^ (y >> 7)) & 0x00AA00AAu;  y = y ^ t ^ (t << 7);
        t = (x ^ (x >> 14)) & 0x0000CCCCu; x = x ^ t ^ (t << 14);
        t = (y ^ (y >> 14)) & 0x0000CCCCu; y = y ^ t ^ (t << 14);
        t = (x ^ (y << 4)) & 0xF0F0F0F0u;  x ^= t; y ^= t >> 4;
        qb[2 * b] = x;
        qb[2 * b + 1] = y;
    }
}

// plane words of 32 byte codes
__device__ __forceinline__ void bytes_to_words(const uint32_t (&qb)[8], int out_bits, uint32_t (&words)[8]) {
    if (out_bits > 2) {
        bytes_to_words_t(qb, words);
        return;
    }
#pragma unroll
    for (int tb = 0; tb < 8; tb++) {
        uint32_t wv = 0;
        if (tb < out_bits) {
#pragma unroll
            for (int qq = 0; qq < 8; qq++) wv |= byte_bits_to_nibble(qb[qq], tb) << (4 * qq);
        }
        words[tb] = wv;
    }
}

// 32 accumulators of row m, columns nb..nb+31 (lc = tile-local column of nb) ->
// plane words: words[t] bit i = bit t of q(column nb + i), t < out_bits.
// Residual requantisation of a 32-column chunk of row m (reading R24):
// q = clamp(floor((alpha*y + beta + rho*z) / S)), z = int32 shortcut or a packed code.
__device__ __forceinline__ void residual_chunk_bytes(const uint32_t (&acc)[32], int m, int nb, const Geom& g,
                                                     const Epi& e, uint32_t (&qb)[8]) {
#pragma unroll
    for (int i = 0; i < 8; i++) qb[i] = 0;
    if (m >= g.M) return;
    const int Nw = (g.N + 127) / 128 * 4;
    uint32_t zw[8];
    if (e.res_bits > 0) {
        const uint32_t* zp = reinterpret_cast<const uint32_t*>(e.res) + (long long)m * e.res_bits * Nw + nb / 32;
#pragma unroll
        for (int t = 0; t < 8; t++) zw[t] = t < e.res_bits ? __ldg(zp + (long long)t * Nw) : 0u;
    }
    const int32_t* zr = reinterpret_cast<const int32_t*>(e.res) + (long long)m * g.N + nb;
#pragma unroll
    for (int g8 = 0; g8 < 4; g8++) {  // 8 columns at a time (register pressure)
        int32_t z[8];
        if (e.res_bits > 0) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                uint32_t code = 0;
#pragma unroll
                for (int t = 0; t < 8; t++) code |= ((zw[t] >> (8 * g8 + i)) & 1u) << t;
                z[i] = (int32_t)code;
            }
        } else if ((g.N & 3) == 0 && nb + 8 * g8 + 8 <= g.N) {
            const int4 a = __ldg(reinterpret_cast<const int4*>(zr + 8 * g8));
            const int4 b = __ldg(reinterpret_cast<const int4*>(zr + 8 * g8 + 4));
            z[0] = a.x; z[1] = a.y; z[2] = a.z; z[3] = a.w; z[4] = b.x; z[5] = b.y; z[6] = b.z; z[7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; i++) z[i] = nb + 8 * g8 + i < g.N ? __ldg(zr + 8 * g8 + i) : 0;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int n = nb + 8 * g8 + i;
            uint32_t q = 0;
            if (n < g.N) {
                const long long r = e.rho ? __ldg(e.rho + n) : 1;
                q = quantise_v(e, (long long)epi_alpha(e, n) * (int32_t)acc[8 * g8 + i] + epi_beta(e, n) + r * z[i]);
            }
            qb[2 * g8 + (i >> 2)] |= q << (8 * (i & 3));
        }
    }
}

// Residual table row (kTabResidual, built once per N tile like the threshold rows): [5] alpha,
// [6] beta, [7] rho of column n; padding columns give q = 0 through alpha = beta = rho = 0.
__device__ __forceinline__ void build_residual_row(int32_t* row, int n, int N, const Epi& e) {
    const bool in = n < N;
    *reinterpret_cast<int4*>(row) = make_int4(0, 0, 0, 0);
    *reinterpret_cast<int4*>(row + 4) =
        make_int4(0, in ? epi_alpha(e, n) : 0, in ? epi_beta(e, n) : 0, in ? (e.rho ? __ldg(e.rho + n) : 1) : 0);
}

// Residual requantisation of a 32-column chunk of row m from the residual table (reading R24):
// v = alpha*y + beta + rho*z in 64 bits, then q = clamp(floor(v / S), 0, Q) with one float
// estimate and one correction (v < Q*S < 2^32 in range and q <= 255, so the estimate is off by at
// most one); packed shortcut codes come out of their planes with words_to_bytes_t.
__device__ __forceinline__ void residual_chunk_bytes_tab(const uint32_t (&acc)[32], int m, int nb, int lc,
                                                         const Geom& g, const Epi& e, const int32_t* tab,
                                                         uint32_t (&qb)[8]) {
#pragma unroll
    for (int i = 0; i < 8; i++) qb[i] = 0;
    if (m >= g.M) return;
    const int Nw = (g.N + 127) / 128 * 4;
    uint32_t zb[8];
    const bool packed = e.res_bits > 0;
    if (packed) {
        const uint32_t* zp = reinterpret_cast<const uint32_t*>(e.res) + (long long)m * e.res_bits * Nw + nb / 32;
        uint32_t zw[8];
#pragma unroll
        for (int t = 0; t < 8; t++) zw[t] = t < e.res_bits ? __ldg(zp + (long long)t * Nw) : 0u;
        words_to_bytes_t(zw, zb);
    }
    const int32_t* zr = reinterpret_cast<const int32_t*>(e.res) + (long long)m * g.N + nb;
    const long long QS = (long long)e.qmax * e.S;
    const uint32_t S = (uint32_t)e.S, Q = (uint32_t)e.qmax;
#pragma unroll
    for (int g8 = 0; g8 < 4; g8++) {  // 8 columns at a time (register pressure)
        int32_t z[8];
        if (packed) {
#pragma unroll
            for (int i = 0; i < 8; i++) z[i] = (int32_t)((zb[2 * g8 + (i >> 2)] >> (8 * (i & 3))) & 0xFFu);
        } else if ((g.N & 3) == 0 && nb + 8 * g8 + 8 <= g.N) {
            const int4 a = __ldg(reinterpret_cast<const int4*>(zr + 8 * g8));
            const int4 b = __ldg(reinterpret_cast<const int4*>(zr + 8 * g8 + 4));
            z[0] = a.x; z[1] = a.y; z[2] = a.z; z[3] = a.w; z[4] = b.x; z[5] = b.y; z[6] = b.z; z[7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; i++) z[i] = nb + 8 * g8 + i < g.N ? __ldg(zr + 8 * g8 + i) : 0;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int4 h = *reinterpret_cast<const int4*>(tab + (lc + 8 * g8 + i) * kTabStride + 4);
            const long long v = (long long)h.y * (int32_t)acc[8 * g8 + i] + h.z + (long long)h.w * z[i];
            uint32_t q;
            if (v < 0) {
                q = 0;
            } else if (v >= QS) {
                q = Q;
            } else {
                const uint32_t v32 = (uint32_t)v;
                q = __float2uint_rz(__uint2float_rn(v32) * e.invS);
                const int32_t r = (int32_t)(v32 - q * S);
                q = r < 0 ? q - 1 : (r >= (int32_t)S ? q + 1 : q);
            }
            qb[2 * g8 + (i >> 2)] |= q << (8 * (i & 3));
        }
    }
}

// RES: compile the residual branch (kTabResidual) in -- only the residual kernel instances,
// so the others keep their register allocation (the residual code cost the 2-CTA kernel
// ~100 bytes of spills per thread when always present)
template <bool RES = false>
__device__ __forceinline__ void requant_chunk(const uint32_t (&acc)[32], int nb, int lc, const Geom& g,
                                              const Epi& e, const int32_t* tab, int tab_mode,
                                              uint32_t (&words)[8], int m = 0) {
    if (tab_mode == kTabQ3) {
        requant_chunk_words_q3(acc, tab, lc, words[0], words[1]);
        return;
    }
    uint32_t qb[8];
#pragma unroll
    for (int i = 0; i < 8; i++) qb[i] = 0;
    if (RES) {
        residual_chunk_bytes(acc, m, nb, g, e, qb);
    } else if (tab_mode == kTabHybrid) {
        const uint32_t S = (uint32_t)e.S, Q = (uint32_t)e.qmax;
#pragma unroll
        for (int i = 0; i < 32; i++)
            qb[i >> 2] |= requant_hybrid(tab + (lc + i) * kTabStride, (int32_t)acc[i], S, e.invS, Q) << (8 * (i & 3));
    } else {
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int n = nb + i;
            uint32_t qv = 0;
            if (n < g.N) qv = requant(e, (int32_t)acc[i], epi_alpha(e, n), epi_beta(e, n));
            qb[i >> 2] |= qv << (8 * (i & 3));
        }
    }
    bytes_to_words(qb, e.out_bits, words);
}

// Direct (per-thread) stores of one 32-column chunk of row m: int32 row segment, or
// the out_bits plane words.  Used where a TMA store box does not fit (partial conv
// row slabs, the one-CTA kernel's packed output).
template <bool RES = false>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&acc)[32], int m, int nb, int lc, const Geom& g,
                                               const Epi& e, void* Yout, const int32_t* tab, int tab_mode) {
    if (m >= g.M) return;
    if (e.out_bits == 0) {
        int32_t* Y = reinterpret_cast<int32_t*>(Yout) + (long long)m * g.N;
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
        return;
    }
    const int Nw = (g.N + 127) / 128 * 4;
    const int word = nb / 32;
    if (word >= Nw) return;
    uint32_t* o = reinterpret_cast<uint32_t*>(Yout) + (long long)m * e.out_bits * Nw + word;
    uint32_t w[8];
    requant_chunk<RES>(acc, nb, lc, g, e, tab, tab_mode, w, m);
#pragma unroll
    for (int tb = 0; tb < 8; tb++)
        if (tb < e.out_bits) o[(long long)tb * Nw] = w[tb];
}

// zero the packed padding words [w_from, Nw) of row m (direct stores)
__device__ __forceinline__ void zero_pad_words(int m, int w_from, const Geom& g, const Epi& e, void* Yout) {
    if (m >= g.M) return;
    const int Nw = (g.N + 127) / 128 * 4;
    uint32_t* o = reinterpret_cast<uint32_t*>(Yout) + (long long)m * e.out_bits * Nw;
    for (int tb = 0; tb < e.out_bits; tb++)
        for (int w = w_from; w < Nw; w++) o[(long long)tb * Nw + w] = 0u;
}

// ---- TMA-store staging (one warp = 32 output rows; lane = row)
// int32: a 32 x 32 block in the SWIZZLE_128B layout of a {32 cols, 32 rows} box:
// 16-byte chunk j of row r at r*128 + ((j ^ (r & 7)) * 16): conflict-free st.shared.v4.
__device__ __forceinline__ void stage_int32_chunk(const uint32_t (&acc)[32], uint8_t* stg, int lane) {
    uint8_t* row = stg + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; j++)
        *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) =
            make_uint4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
}
// Coalesced write-back of a staged 32 x 32 int32 block (rows row0.., columns col0..):
// lane l moves 16-byte piece (l & 7) of rows 4i + (l >> 3), so every st.global.v4
// instruction writes four whole 128-byte row segments.  Rows >= row_end and columns
// >= N are not written.  Requires N % 4 == 0.
__device__ __forceinline__ void writeback_int32_block(const uint8_t* stg, int lane, int32_t* Y, int row0,
                                                      int row_end, int col0, int N) {
    const int j = lane & 7;
    const int col = col0 + 4 * j;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int r = 4 * i + (lane >> 3);
        const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 128 + ((j ^ (r & 7)) << 4));
        if (row0 + r < row_end && col < N)
            *reinterpret_cast<uint4*>(Y + (long long)(row0 + r) * N + col) = v;
    }
}
// Coalesced write-back of a staged packed box [32 rows][bits][nwb words] to
// out[m][t][w0 .. w0 + nwb) (clipped at Nw and row_end); lane handles 16-byte pieces.
__device__ __forceinline__ void writeback_packed_block(const uint32_t* stg, int lane, uint32_t* out, int row0,
                                                       int row_end, int w0, int Nw, int bits, int nwb) {
    const int per_row = bits * nwb / 4;  // 16-byte pieces per row
    const int total = 32 * per_row;
    for (int i = lane; i < total; i += 32) {
        const int r = i / per_row, pc = i - r * per_row;
        const int t = (pc * 4) / nwb, w = (pc * 4) - t * nwb;
        if (row0 + r < row_end && w0 + w < Nw)
            *reinterpret_cast<uint4*>(out + ((long long)(row0 + r) * bits + t) * Nw + w0 + w) =
                *reinterpret_cast<const uint4*>(stg + r * bits * nwb + t * nwb + w);
    }
}
// packed: a {nwb words, bits, 32 rows} box, dense [row][plane][nwb] uint32
__device__ __forceinline__ void stage_words(const uint32_t (&w)[8], int bits, int nwb, int wi, uint32_t* stg,
                                            int lane) {
    uint32_t* row = stg + lane * bits * nwb + wi;
#pragma unroll
    for (int tb = 0; tb < 8; tb++)
        if (tb < bits) row[tb * nwb] = w[tb];
}

}  // namespace tc
}  // namespace apnn
