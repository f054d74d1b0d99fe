// conv_halo.cu -- APConv (convolution as implicit GEMM) with filter-tap
// reuse: the "halo" kernel behind apnn_conv2d_prepared_i8.
//
// The per-tap implicit GEMM of gemm_tc.cu decodes every input pixel's bit planes once PER
// FILTER TAP (9x for a 3x3 layer) and hands a k-block to the MMA per tap.  Here a CTA owns a
// 16 x 8 tile of output pixels and, per 128-channel chunk, decodes the tile's input window
// (halo) ONCE from the packed planes into int8 rows in shared memory (the operand-side bit
// combination, PAPER.md:1426-1429 applied to the operand, as in gemm_tc.cu), laid out as one
// copy per (row phase rho = r mod stride, column tap s):
//
//     copy[rho][s][j][tw] = x[b][stride*hh + rho - pad][stride*(w0 + tw) + s - pad]
//
// where row j of the copy is "tall" row v0 + j = b*Hv + hh of the batch seen as one image of
// Hv = Ho + (R-1)/stride rows per image (rows hh >= Ho are separators whose outputs are
// discarded).  Filter tap (r, s) of output pixel (v0 + hv, w0 + tw) is then copy row
// hv + r/stride of copy (r mod stride, s): the A operand of tap (r, s) is the 128-row window
// of that copy starting (r / stride) 8-row core-matrix groups in -- a descriptor offset, no
// data movement.  All R*S taps of the chunk run back to back on the tensor core from one
// decode (R*S*Cc/32 MMAs per hand-off instead of Cc/32).
//
// Pair kernel (cta_group::2): the two CTAs of a cluster hold two 128-pixel tiles (M = 256)
// and half of the N tile's weight rows each; prepared int8 weights (apnn_prepare_weights_i8,
// [C_out][R*S*Cp] bytes) arrive by TMA (SWIZZLE_128B); when the whole N tile fits they are
// loaded once and stay resident.  Warp roles per CTA:
//   warps 0-7   decode: (pixel, 32-channel group) units -> int8 copies (K-major, no swizzle)
//   warps 8-15  epilogue (two per TMEM lane quarter): TMEM -> int32 NHWC, or requantise + pack
//               (PAPER.md:1296-1306), optional fused 2x2/2 max pooling (warp shuffles) or
//               residual (reading R24)
//   warp 16     forwards "W stage landed" to CTA 0 (the MMA issuer needs both halves)
//   warp 17     TMA producer of the weight stages
//   warp 18     TMEM allocator; CTA 0 lane 0 issues tcgen05.mma
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_common.cuh"

namespace apnn {
namespace halo {

using namespace tc;

constexpr int TH = 16, TW = 8;  // CTA tile: 16 (tall) output rows x 8 columns = 128 MMA rows
constexpr int DEC_WARPS = 8;
constexpr int DEC_THREADS = DEC_WARPS * 32;
constexpr int EPI0 = DEC_WARPS;
constexpr int EPI_WARPS = 8;
constexpr int FWD_WARP = EPI0 + EPI_WARPS;
constexpr int TMA_WARP = FWD_WARP + 1;
constexpr int MMA_WARP = TMA_WARP + 1;
constexpr int THREADS = (MMA_WARP + 1) * 32;
constexpr int MAX_WS = 40;  // weight stages (resident: all R*S*chunks of the N tile)
// epilogue staging per warp: int32 32 x 32 block (4 KB); packed: mt = 1 two warps share 32 x 68 words
// per quarter (2 x 4352 B), mt = 2 one warp owns 32 x 36 words (4608 B)
constexpr int STG1 = 4352, STG2 = 4608;

struct Params {
    Geom g;
    Epi e;
    void* Y;
    const uint32_t* X;
    const uint8_t* Xraw;  // first layer: raw 8-bit NHWC image (quantised while decoding)
    int raw, qz, qs;      // raw mode, quantisation q = clamp(floor((x - qz) / qs), 0, 2^a_bits - 1)
    int S_raw, C_raw;     // raw mode: the window (S_raw columns x C_raw channels) is one copy row
    int B;
    int Hv, E;            // tall rows per image, extra copy rows (R-1)/stride
    int nrho, ncopy;      // row phases min(stride, R); copies nrho * S
    int crow;             // copy rows (groups of 8 pixels) = TH + E
    int cl;               // copy row bytes: 32 / 64 / 128 (= the UMMA swizzle width; C_in <= 32 / 64 / else)
    int cc8;              // bytes per 8-row swizzle atom = 8 * cl (the descriptor's SBO)
    int smask;            // 16-byte chunk XOR mask of the swizzle: cl / 16 - 1
    int G;                // 32-channel groups decoded per copy row: ceil(min(C_in, 128) / 32)
    int nchunk;           // 128-channel chunks (= CB)
    int ixn;              // input columns a tile touches: stride*(TW-1) + S
    uint32_t copy_bytes, set_bytes;
    int nbuf;             // copy sets (double buffering when it fits)
    int ws, w_resident, nsteps;
    int bn;               // N tile of the pair (each CTA holds bn/2 weight rows)
    int tiles_c, cta_tiles, pair_tiles, n_tiles, num_tiles;
    int tab_mode, pool_fused, Hp, Wp;
    uint32_t tmem_cols;
    int mt, th;           // 128-row sub-tiles per CTA tile (1 or 2) and the tile's tall rows (16 * mt)
    int stg;              // epilogue staging bytes per warp (STG1 / STG2)
    int exp;              // experiment builds only (APNN_DEV): 1 skip decode, 2 skip MMAs, 4 skip epilogue
    unsigned long long* trace;  // experiment builds only: %globaltimer stamps of CTAs 0/1 (APNN_HALO_TRACE)
};
#ifndef APNN_DEV
#define APNN_DEV 0
#endif
constexpr bool kDev = APNN_DEV != 0;
#ifndef APNN_HALO_SLEEP
#define APNN_HALO_SLEEP 2
#endif
// barrier waits: the MMA issuer spins (its wake-up latency is on the critical path), the other
// roles sleep in the try_wait (suspend-time hint) so they do not take the issuer's issue slots
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t ph) {
    if (APNN_HALO_SLEEP == 1) sm100::mbar_wait_sleep(bar, ph);
    else sm100::mbar_wait(bar, ph);
}
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t ph) {
    if (APNN_HALO_SLEEP >= 1) sm100::mbar_wait_sleep(bar, ph);
    else sm100::mbar_wait(bar, ph);
}
constexpr int kTrN = 512;
enum { TR_PROD, TR_FWD, TR_MMA_W, TR_MMA_DONE, TR_DEC_GO, TR_DEC_DONE, TR_MMA_C, TR_EPI_GO, TR_EPI_DONE, TR_MMA_A,
       TR_NEV };
__device__ __forceinline__ void trace(const Params& p, int ev, int i) {
    if (kDev && p.trace && blockIdx.x < 2 && i < kTrN) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles (CTA 0 / CTA 1 clocks differ)
        p.trace[((size_t)blockIdx.x * TR_NEV + ev) * kTrN + i] = t;
    }
}

// ---------------------------------------------------------------- decode
// Work split of the decode warps, fixed for the kernel: thread tid owns 32-channel group gi and
// input column ixo of every tile (units = (gi, ixo) pairs, gi fastest), and walks the copy rows
// jr, jr + jstep, ...  The copies that read column ixo -- copy s at tile column tw where
// stride*tw + s = ixo -- are precomputed as byte offsets, so the per-row work is one pixel
// address, the plane loads, the recombination and the stores.
constexpr int kMaxTg = 8;  // copies one input column feeds: ceil(S / stride) <= 8
struct DecCtx {
    bool active;
    int gi, jr, jstep, iw_rel;
    int ntg;
    uint32_t tg[kMaxTg];  // target offsets: copy s base + tw * cl
};

__device__ __forceinline__ DecCtx make_dec_ctx(const Params& p, int tid) {
    const Geom& g = p.g;
    DecCtx d;
    const int cols = p.G * p.ixn;
    d.jstep = DEC_THREADS / cols;
    d.active = tid < d.jstep * cols;
    const int u = d.active ? tid : 0;
    d.gi = u % p.G;
    const int ixo = (u / p.G) % p.ixn;
    d.jr = u / cols;
    d.iw_rel = ixo - g.pad;
    d.ntg = 0;
#pragma unroll
    for (int q = 0; q < kMaxTg; q++) d.tg[q] = 0;
    for (int sx = 0; sx < g.S; sx++) {
        const int dd = ixo - sx;
        if (dd < 0) break;
        const int tw = dd / g.stride;
        if (tw * g.stride != dd || tw >= TW) continue;
        const uint32_t off = (uint32_t)sx * p.copy_bytes + (uint32_t)tw * p.cl;
#pragma unroll
        for (int q = 0; q < kMaxTg; q++)
            if (q == d.ntg) d.tg[q] = off;
        d.ntg++;
    }
    return d;
}

// Decode one 128-channel chunk of a tile's input window into the copies: the pixel's NB plane
// words are recombined into 32 int8 operand bytes (decode_01 / decode_pm1: the element order of
// tc_common.cuh, which the prepared weights share) and stored into every copy that reads the
// pixel.  Out-of-frame pixels and padded channels are value 0 for every encoding
// (reading R16).  kU rows per round: their loads are all issued first.
template <int NB, bool PM1>
__device__ __forceinline__ void decode_chunk(const Params& p, const DecCtx& d, uint8_t* set, int v0, int w0, int ci) {
    const Geom& g = p.g;
    const int gc = ci * 4 + d.gi;  // 32-channel group = word index inside a plane run
    if (!d.active || gc * 32 >= g.C) return;  // groups past C_in are not read by the MMAs
    constexpr int kU = NB <= 2 ? 4 : 2;
    const uint32_t vm = valid_mask(g.C - gc * 32, 0);
    const int st = g.stride, crow = p.crow, jstep = d.jstep, H = g.H, Hv = p.Hv, B = p.B, pad = g.pad;
    const int iw = st * w0 + d.iw_rel;
    const bool col_in = iw >= 0 && iw < g.W;
    const long long pix_stride = (long long)NB * g.Cw;  // words per pixel record
    const uint32_t* xcol = p.X + (long long)iw * pix_stride + gc;
    const uint32_t smask = p.smask;
    for (int rho = 0; rho < p.nrho; rho++) {
        const uint32_t rbase = (uint32_t)rho * g.S * p.copy_bytes + (uint32_t)d.gi * 32;
        for (int j0 = d.jr; j0 < crow; j0 += kU * jstep) {
            uint32_t pw[kU][NB];
            bool in[kU];
#pragma unroll
            for (int k = 0; k < kU; k++) {
                const int j = j0 + k * jstep;
                const int vr = v0 + j;
                const int b = vr / Hv, hh = vr - b * Hv;
                const int ih = st * hh + rho - pad;
                in[k] = j < crow && col_in && b < B && ih >= 0 && ih < H;
                const uint32_t* src = xcol + ((long long)b * H + ih) * g.W * pix_stride;
#pragma unroll
                for (int t = 0; t < NB; t++) pw[k][t] = in[k] ? __ldg(src + t * g.Cw) : 0u;
            }
#pragma unroll
            for (int k = 0; k < kU; k++) {
                const int j = j0 + k * jstep;
                if (j >= crow) break;
                uint32_t o[8];
                if (PM1) decode_pm1<true>(pw[k][0], in[k] ? vm : 0u, o);  // out of frame: value 0
                else decode_01<NB>(pw[k], o);                              // zero planes decode to 0
                const uint4 lo = make_uint4(o[0], o[1], o[2], o[3]), hi = make_uint4(o[4], o[5], o[6], o[7]);
                // K-major swizzled operand rows (SWIZZLE_32B/64B/128B, atoms of 8 rows x cl bytes):
                // chunk c of a row at byte offset A lands at A ^ (((A >> 7) & smask) << 4)
                const uint32_t row = rbase + (uint32_t)j * p.cc8;
#pragma unroll
                for (int q = 0; q < kMaxTg; q++) {
                    if (q >= d.ntg) break;
                    const uint32_t a = row + d.tg[q], a1 = a + 16;
                    *reinterpret_cast<uint4*>(set + (a ^ (((a >> 7) & smask) << 4))) = lo;
                    *reinterpret_cast<uint4*>(set + (a1 ^ (((a1 >> 7) & smask) << 4))) = hi;
                }
            }
        }
    }
}

template <bool PM1>
__device__ __forceinline__ void decode_chunk_any(const Params& p, const DecCtx& d, uint8_t* set, int v0, int w0,
                                                 int ci) {
    if (PM1) {
        decode_chunk<1, true>(p, d, set, v0, w0, ci);
        return;
    }
    switch (p.g.a_bits) {
    case 1: decode_chunk<1, false>(p, d, set, v0, w0, ci); break;
    case 2: decode_chunk<2, false>(p, d, set, v0, w0, ci); break;
    case 3: decode_chunk<3, false>(p, d, set, v0, w0, ci); break;
    case 4: decode_chunk<4, false>(p, d, set, v0, w0, ci); break;
    case 5: decode_chunk<5, false>(p, d, set, v0, w0, ci); break;
    case 6: decode_chunk<6, false>(p, d, set, v0, w0, ci); break;
    case 7: decode_chunk<7, false>(p, d, set, v0, w0, ci); break;
    default: decode_chunk<8, false>(p, d, set, v0, w0, ci); break;
    }
}

// ---------------------------------------------------------------- first layer
// Raw mode (the first layer, reading R23): the layer reads the 8-bit image
// and quantises it while decoding, q = clamp(floor((x - z) / s), 0, 2^a_bits - 1) through a
// 256-entry table; the contraction runs over taps r (rows) with K = the S x C_in window of one
// input row, which is contiguous in NHWC.  A unit is one copy row (rho, j, tw): its window's
// codes land at the recombination's element positions (byte 4*(k%8) + (k%32)/8 of group k/32,
// the order of the prepared weights, viewed as C_out*R rows of S*C_in).  Out-of-frame pixels are
// code 0 (zero padding of the quantised activations, as the oracle's first layer).
template <int SR, int CR>
__device__ __forceinline__ void decode_raw_fixed(const Params& p, uint8_t* set, int v0, int w0, const uint8_t* qtab,
                                                 int tid) {
    constexpr int KW = SR * CR;
    constexpr int GW = (KW + 31) / 32;  // 32-byte groups of the row
    const Geom& g = p.g;
    const int st = g.stride, crow = p.crow, Hv = p.Hv, H = g.H, W = g.W, pad = g.pad;
    const int units = p.nrho * crow * TW;
    const uint32_t smask = p.smask;
    for (int u = tid; u < units; u += DEC_THREADS) {
        const int tw = u & (TW - 1);
        const int rest = u >> 3;
        const int rho = rest / crow, j = rest - rho * crow;
        const int vr = v0 + j;
        const int b = vr / Hv, hh = vr - b * Hv;
        const int ih = st * hh + rho - pad;
        const int iw0 = st * (w0 + tw) - pad;
        const bool rowin = b < p.B && ih >= 0 && ih < H;
        const uint8_t* src = p.Xraw + ((long long)(b * H + ih) * W + iw0) * CR;
        uint32_t wv[8 * GW];
#pragma unroll
        for (int i = 0; i < 8 * GW; i++) wv[i] = 0u;
#pragma unroll
        for (int sx = 0; sx < SR; sx++) {
            const bool in = rowin && iw0 + sx >= 0 && iw0 + sx < W;
#pragma unroll
            for (int c = 0; c < CR; c++) {
                const int k = sx * CR + c;
                const uint32_t code = in ? (uint32_t)qtab[__ldg(src + k)] : 0u;
                wv[8 * (k / 32) + (k % 8)] |= code << (8 * ((k % 32) / 8));
            }
        }
        const uint32_t row = (uint32_t)rho * p.copy_bytes + (uint32_t)j * p.cc8 + (uint32_t)tw * p.cl;
#pragma unroll
        for (int gi = 0; gi < GW; gi++) {
            const uint32_t a = row + (uint32_t)gi * 32, a1 = a + 16;
            *reinterpret_cast<uint4*>(set + (a ^ (((a >> 7) & smask) << 4))) =
                make_uint4(wv[8 * gi], wv[8 * gi + 1], wv[8 * gi + 2], wv[8 * gi + 3]);
            *reinterpret_cast<uint4*>(set + (a1 ^ (((a1 >> 7) & smask) << 4))) =
                make_uint4(wv[8 * gi + 4], wv[8 * gi + 5], wv[8 * gi + 6], wv[8 * gi + 7]);
        }
    }
}

// any window (S_raw * C_raw <= 128): codes stored byte by byte, the rest of the row's groups zeroed
__device__ __forceinline__ void decode_raw_any(const Params& p, uint8_t* set, int v0, int w0, const uint8_t* qtab,
                                               int tid) {
    const Geom& g = p.g;
    const int SR = p.S_raw, CR = p.C_raw, KW = SR * CR, GW = (KW + 31) / 32;
    const int st = g.stride, crow = p.crow, Hv = p.Hv, H = g.H, W = g.W, pad = g.pad;
    const int units = p.nrho * crow * TW;
    const uint32_t smask = p.smask;
    for (int u = tid; u < units; u += DEC_THREADS) {
        const int tw = u & (TW - 1);
        const int rest = u >> 3;
        const int rho = rest / crow, j = rest - rho * crow;
        const int vr = v0 + j;
        const int b = vr / Hv, hh = vr - b * Hv;
        const int ih = st * hh + rho - pad;
        const int iw0 = st * (w0 + tw) - pad;
        const bool rowin = b < p.B && ih >= 0 && ih < H;
        const uint8_t* src = p.Xraw + ((long long)(b * H + ih) * W + iw0) * CR;
        const uint32_t row = (uint32_t)rho * p.copy_bytes + (uint32_t)j * p.cc8 + (uint32_t)tw * p.cl;
        for (int k = 0; k < GW * 32; k++) {
            uint32_t code = 0;
            if (k < KW) {
                const int sx = k / CR;
                if (rowin && iw0 + sx >= 0 && iw0 + sx < W) code = qtab[__ldg(src + k)];
            }
            const uint32_t a = row + (uint32_t)(k / 32) * 32 + (uint32_t)(4 * (k % 8) + (k % 32) / 8);
            set[a ^ (((a >> 7) & smask) << 4)] = (uint8_t)code;
        }
    }
}

__device__ __forceinline__ void tile_origin(const Params& p, int tile, uint32_t rank, int& ct, int& v0, int& w0,
                                            int& n0) {
    const int pt = tile % p.pair_tiles, nt = tile / p.pair_tiles;
    ct = 2 * pt + (int)rank;
    const int rb = ct / p.tiles_c, cb = ct - rb * p.tiles_c;
    v0 = rb * p.th;
    w0 = cb * TW;
    n0 = nt * p.bn;
}

// MMA issuer (one thread of CTA 0).  Its instruction stream is the critical path (an M=256
// N=64 K=32 MMA runs in ~32 cycles), so everything it needs is loaded into registers before the
// tile loop: with RST = 9 (3x3 filters) the tap loop is unrolled and the taps' A offsets are
// registers; descriptors advance by 64-bit adds; ring counters are incremental.
template <int RST, int MT, bool A_PM1, bool W_PM1>
__device__ __forceinline__ void mma_issuer(const Params& p, const uint32_t* sTap, uint8_t* sCopy, uint8_t* sW,
                                        uint64_t* w_ready, uint64_t* w_empty, uint64_t* c_full, uint64_t* c_empty,
                                        uint64_t* a_full, uint64_t* a_empty, uint32_t tmem, int my_tiles) {
    using namespace sm100;
    const int RS = RST ? RST : p.g.RS;
    const int nchunk = p.nchunk, nbuf = p.nbuf, ws = p.ws, bn = p.bn, C = p.g.C;
    const bool resident = p.w_resident != 0;
    const bool skip_mma = kDev && (p.exp & 2);
    const uint32_t idesc = idesc_i8(256, bn, A_PM1, W_PM1);
    const uint64_t swz = p.cl == 128 ? 2ull : (p.cl == 64 ? 4ull : 6ull);  // descriptor layout type
    const uint64_t ad0 = (umma_desc_sw128(smem_u32(sCopy), (uint32_t)p.cc8) & ~(7ull << 61)) | (swz << 61);
    const uint64_t bd0 = umma_desc_sw128(smem_u32(sW), 1024);
    const uint32_t set16 = p.set_bytes >> 4, wst16 = ((uint32_t)(bn / 2) * 128u) >> 4;
    constexpr int mt = MT;
    const uint32_t sub16 = (uint32_t)p.cc8;  // 16 copy rows (one 8-row swizzle atom each) = 16 * cc8 bytes, in 16-B units
    uint32_t toff[RST ? RST : 1];
    if (RST) {
#pragma unroll
        for (int rs = 0; rs < (RST ? RST : 1); rs++) toff[rs] = sTap[rs];
    }
    int s = 0, cb = 0;
    uint32_t wph = 0, cph = 0;
    for (int k = 0; k < my_tiles; k++) {
        const int buf = k & 1;
        const uint32_t dtm = tmem + (uint32_t)(buf * mt * bn);
        mma_wait(&a_empty[buf], ((k >> 1) & 1) ^ 1);
        trace(p, TR_MMA_A, k);
        tc_fence_after();
        uint32_t acc = 0;
        for (int ci = 0; ci < nchunk; ci++) {
            mma_wait(&c_full[cb], cph);
            trace(p, TR_MMA_C, k * nchunk + ci);
            tc_fence_after();
            const int crem = C - ci * 128;
            const int nkk = crem >= 128 ? 4 : (crem + 31) / 32;
            const uint64_t ads = ad0 + (uint64_t)((uint32_t)cb * set16);
            if (resident) s = ci * RS;
            const int rs_end = (kDev && (p.exp & 32) && k > 0) ? 0 : RS;
#pragma unroll
            for (int rs = 0; rs < rs_end; rs++) {
                if (!resident || k == 0) {
                    mma_wait(&w_ready[s], resident ? 0u : wph);
                    tc_fence_after();
                }
                const uint64_t ad = ads + (RST ? toff[RST ? rs : 0] : sTap[rs]);
                const uint64_t bd = bd0 + (uint64_t)((uint32_t)s * wst16);
                if (!skip_mma) {
                    mma2_i8_ss(dtm, ad, bd, idesc, acc);
                    if (nkk > 1) mma2_i8_ss(dtm, ad + 2, bd + 2, idesc, 1u);
                    if (nkk > 2) mma2_i8_ss(dtm, ad + 4, bd + 4, idesc, 1u);
                    if (nkk > 3) mma2_i8_ss(dtm, ad + 6, bd + 6, idesc, 1u);
                    if (mt > 1) {  // second 128-row sub-tile: the A window 16 copy rows further, its own accumulator
                        const uint64_t ad1 = ad + sub16;
                        const uint32_t d1 = dtm + (uint32_t)bn;
                        mma2_i8_ss(d1, ad1, bd, idesc, acc);
                        if (nkk > 1) mma2_i8_ss(d1, ad1 + 2, bd + 2, idesc, 1u);
                        if (nkk > 2) mma2_i8_ss(d1, ad1 + 4, bd + 4, idesc, 1u);
                        if (nkk > 3) mma2_i8_ss(d1, ad1 + 6, bd + 6, idesc, 1u);
                    }
                }
                acc = 1u;
                if (!resident) {
                    mma2_commit_mc(&w_empty[s], 0x3);
                    if (++s == ws) { s = 0; wph ^= 1u; }
                } else {
                    s++;
                }
            }
            trace(p, TR_MMA_DONE, k * nchunk + ci);
            mma2_commit_mc(&c_empty[cb], 0x3);
            if (++cb == nbuf) { cb = 0; cph ^= 1u; }
        }
        mma2_commit_mc(&a_full[buf], 0x3);
    }
}

// ================================================================ kernel
template <bool A_PM1, bool W_PM1, bool RES, bool RAW = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    halo_kernel(const __grid_constant__ CUtensorMap tmapW, const Params p) {
    using namespace sm100;
    extern __shared__ __align__(1024) uint8_t smem[];
    const Geom& g = p.g;
    const uint32_t WSTAGE = (uint32_t)(p.bn / 2) * 128u;
    uint8_t* sW = smem;                                             // ws x (bn/2 rows x 128 B), SWIZZLE_128B
    uint8_t* sCopy = sW + (size_t)p.ws * WSTAGE;                    // nbuf x set_bytes
    uint8_t* sStg = sCopy + (size_t)p.nbuf * p.set_bytes;           // EPI_WARPS x p.stg
    int32_t* sTab = reinterpret_cast<int32_t*>(sStg + EPI_WARPS * p.stg);  // bn x kTabStride
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + p.bn * kTabStride);
    uint64_t* w_full = bars;                  // [MAX_WS] local TMA completion
    uint64_t* w_empty = w_full + MAX_WS;      // [MAX_WS] local, MMA commit (multicast)
    uint64_t* w_ready = w_empty + MAX_WS;     // [MAX_WS] CTA 0: both halves landed (2 forwards)
    uint64_t* c_full = w_ready + MAX_WS;      // [2] CTA 0: copies written (2 x DEC_WARPS)
    uint64_t* c_empty = c_full + 2;           // [2] local, MMA commit (multicast)
    uint64_t* a_full = c_empty + 2;           // [2] local, MMA commit (multicast)
    uint64_t* a_empty = a_full + 2;           // [2] CTA 0: 2 x 4 epilogue warps
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(a_empty + 2);  // [4] + tap table [RS]

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (warp == TMA_WARP && lane == 0) {
        tma_prefetch(&tmapW);
        for (int s = 0; s < p.ws; s++) {
            mbar_init(&w_full[s], 1);
            mbar_init(&w_empty[s], 1);
            mbar_init(&w_ready[s], 2);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&c_full[i], 2 * DEC_WARPS);
            mbar_init(&c_empty[i], 1);
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 2 * EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == MMA_WARP) tmem_alloc2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const int my_tiles = p.num_tiles > cid ? (p.num_tiles - cid + ncl - 1) / ncl : 0;
    // Programmatic dependent launch (the host launches with programmatic stream serialization):
    // the prologue above -- barrier init, TMEM allocation, tensor-map prefetch -- overlaps the
    // previous kernel's tail; activations, weights and outputs are touched only after the previous
    // grid has completed and its memory is visible.  The next kernel may be scheduled as soon as
    // every CTA of this one is past this point (its CTAs start on SMs this grid has left).
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // The single-thread roles keep their whole warp converged in the loop (every lane waits on
    // the barriers, lane 0 issues): a lone lane spinning while its 31 siblings sit at the final
    // __syncthreads was measured to cost ~0.4 us per loop iteration (divergent-path scheduling).
    if (warp == TMA_WARP) {
        // ------------------------------------------------ weight producer
        const int nrow0 = (int)rank * (p.bn / 2);
        if (p.w_resident) {
            if (lane == 0) {
                for (int s = 0; s < p.nsteps; s++) {
                    const int ci = s / g.RS, rs = s - ci * g.RS;
                    mbar_arrive_expect_tx(&w_full[s], WSTAGE);
                    tma_load_2d(sW + (size_t)s * WSTAGE, &tmapW, &w_full[s], (rs * g.CB + ci) * 128, nrow0);
                }
            }
            __syncwarp();
        } else {
            int it = 0;
            for (int k = 0; k < my_tiles; k++) {
                const int tile = cid + k * ncl;
                const int n0 = (tile / p.pair_tiles) * p.bn;
                for (int st = 0; st < p.nsteps; st++, it++) {
                    const int ci = st / g.RS, rs = st - ci * g.RS;
                    const int s = it % p.ws;
                    const uint32_t ph = (uint32_t)(it / p.ws) & 1u;
                    role_wait(&w_empty[s], ph ^ 1u);
                    if (lane == 0) {
                        trace(p, TR_PROD, it);
                        mbar_arrive_expect_tx(&w_full[s], WSTAGE);
                        tma_load_2d(sW + (size_t)s * WSTAGE, &tmapW, &w_full[s], (rs * g.CB + ci) * 128, n0 + nrow0);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == FWD_WARP) {
        // ------------------------------------------------ "stage landed" -> CTA 0
        const uint32_t ready0 = mapa(smem_u32(w_ready), 0);
        const int total = p.w_resident ? p.nsteps : my_tiles * p.nsteps;
        for (int it = 0; it < total; it++) {
            const int s = it % p.ws;
            role_wait(&w_full[s], (uint32_t)(it / p.ws) & 1u);
            if (lane == 0) {
                trace(p, TR_FWD, it);
                mbar_arrive_cluster(ready0 + 8u * (uint32_t)s);
            }
            __syncwarp();
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------ MMA issuer (CTA 0)
        // One thread issues every MMA, so its instruction stream is the critical path (an M=256
        // N=64 K=32 MMA runs in ~32 cycles): all loop constants live in registers, the A offset
        // of each tap comes from a table built once, descriptors advance by plain adds, and the
        // ring counters are incremental (no divisions, no parameter reloads per MMA).
        if (rank == 0) {
            uint32_t* sTap = tmem_holder + 4;  // [RS] A-operand offsets of the taps (16-byte units)
            for (int rs = lane; rs < g.RS; rs += 32) {
                const int r = rs / g.S, sx = rs - r * g.S;
                sTap[rs] = ((uint32_t)((r % g.stride) * g.S + sx) * p.copy_bytes + (uint32_t)(r / g.stride) * p.cc8) >> 4;
            }
            __syncwarp();
            if (lane == 0) {
                // one instantiation per (3x3 or not, sub-tiles): the single issuing thread runs
                // straight-line code without branches for the other shapes
                if (g.RS == 9 && p.mt == 2)
                    mma_issuer<9, 2, A_PM1, W_PM1>(p, sTap, sCopy, sW, w_ready, w_empty, c_full, c_empty, a_full,
                                                   a_empty, tmem, my_tiles);
                else if (g.RS == 9)
                    mma_issuer<9, 1, A_PM1, W_PM1>(p, sTap, sCopy, sW, w_ready, w_empty, c_full, c_empty, a_full,
                                                   a_empty, tmem, my_tiles);
                else if (p.mt == 2)
                    mma_issuer<0, 2, A_PM1, W_PM1>(p, sTap, sCopy, sW, w_ready, w_empty, c_full, c_empty, a_full,
                                                   a_empty, tmem, my_tiles);
                else
                    mma_issuer<0, 1, A_PM1, W_PM1>(p, sTap, sCopy, sW, w_ready, w_empty, c_full, c_empty, a_full,
                                                   a_empty, tmem, my_tiles);
            }
        }
    } else if (warp < DEC_WARPS) {
        // ------------------------------------------------ decode
        const DecCtx dctx = make_dec_ctx(p, threadIdx.x);
        const uint32_t c_full0 = mapa(smem_u32(c_full), 0);
        uint8_t* qtab = reinterpret_cast<uint8_t*>(tmem_holder + 4 + 64);  // raw mode: 256-entry code table
        if (RAW) {
            const int x = threadIdx.x;  // DEC_THREADS == 256
            const int v = x - p.qz;
            const int qv = v < 0 ? 0 : v / p.qs;
            const int qmax = (1 << g.a_bits) - 1;
            qtab[x] = (uint8_t)(qv > qmax ? qmax : qv);
            named_bar_sync(6, DEC_THREADS);
        }
        int q = 0;
        for (int k = 0; k < my_tiles; k++) {
            int ct, v0, w0, n0;
            tile_origin(p, cid + k * ncl, rank, ct, v0, w0, n0);
            for (int ci = 0; ci < p.nchunk; ci++, q++) {
                const int cb = q % p.nbuf;
                role_wait(&c_empty[cb], ((uint32_t)(q / p.nbuf) & 1u) ^ 1u);
                if (threadIdx.x == 0) trace(p, TR_DEC_GO, q);
                if (ct < p.cta_tiles && !(kDev && (p.exp & 1))) {
                    uint8_t* set = sCopy + (size_t)cb * p.set_bytes;
                    if (RAW) {
                        if (p.S_raw == 7 && p.C_raw == 3) decode_raw_fixed<7, 3>(p, set, v0, w0, qtab, threadIdx.x);
                        else if (p.S_raw == 11 && p.C_raw == 3) decode_raw_fixed<11, 3>(p, set, v0, w0, qtab, threadIdx.x);
                        else decode_raw_any(p, set, v0, w0, qtab, threadIdx.x);
                    } else {
                        decode_chunk_any<A_PM1>(p, dctx, set, v0, w0, ci);
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(c_full0 + 8u * (uint32_t)cb);
                if (threadIdx.x == 0) trace(p, TR_DEC_DONE, q);
            }
        }
    } else if (warp < FWD_WARP) {
        // ------------------------------------------------ epilogue
        // 8 warps: warp EPI0 + e reads TMEM lane quarter e & 3 (tile rows 32*(e&3)..) and takes
        // every other 32-column chunk (half e >> 2), so each SM sub-partition runs two epilogue
        // warps.  Packed output: both warps of a quarter stage their plane words in that
        // quarter's [row][plane][nwt (+4 pad)] buffer, meet on a named barrier, and each thread
        // stores whole 16-byte pieces of its own row (no shuffles, no divisions).
        const int e8 = warp - EPI0;
        const int qw = e8 & 3, half = e8 >> 2;
        // mt = 1: the two warps of a quarter split the columns (half); mt = 2: warp half takes
        // sub-tile `half` (tile rows 128 * half + ...) with all the columns, its own staging
        const int mt = p.mt, sub = mt > 1 ? half : 0, cstep = mt > 1 ? 32 : 64, c0 = mt > 1 ? 0 : half * 32;
        const int t = sub * 128 + qw * 32 + lane;  // tile row = hv * 8 + tw (TMEM lane qw * 32 + lane)
        const int et = threadIdx.x - EPI0 * 32;
        const uint32_t tmem_lane = tmem + ((uint32_t)(qw * 32) << 16);
        const uint32_t a_empty0 = mapa(smem_u32(a_empty), 0);
        const int ob = p.e.out_bits;
        const int Nw = (g.N + 127) / 128 * 4;
        const int bn = p.bn;
        uint8_t* stg_q = sStg + qw * (2 * p.stg) + (mt > 1 ? half * p.stg : 0);  // packed staging
        uint8_t* stg_w = sStg + qw * (2 * p.stg) + half * p.stg;  // int32: this warp's own 32 x 32 block
        int cur_n0 = -1;
        for (int k = 0; k < my_tiles; k++) {
            int ct, v0, w0, n0;
            tile_origin(p, cid + k * ncl, rank, ct, v0, w0, n0);
            if ((p.tab_mode == kTabQ3 || p.tab_mode == kTabHybrid || (RES && p.tab_mode == kTabResidual)) &&
                n0 != cur_n0) {
                named_bar_sync(1, 256);
                for (int c = et; c < bn; c += 256) {
                    if (RES && p.tab_mode == kTabResidual) build_residual_row(sTab + c * kTabStride, n0 + c, g.N, p.e);
                    else build_threshold_row(sTab + c * kTabStride, n0 + c, g.N, p.e);
                }
                named_bar_sync(1, 256);
                cur_n0 = n0;
            }
            const int hv = t >> 3, tw = t & 7;
            const int vr = v0 + hv;
            const int b = vr / p.Hv, ho = vr - b * p.Hv, wo = w0 + tw;
            const bool valid = ct < p.cta_tiles && b < p.B && ho < g.Ho && wo < g.Wo;
            const int m = valid ? (b * g.Ho + ho) * g.Wo + wo : g.M;
            // packed words of this tile per row: the bn columns, plus the N padding on the last tile
            const int nwt = (n0 + bn >= g.N) ? Nw - n0 / 32 : bn / 32;
            const int rstride = ob * nwt + 4;  // staged row stride in words (16-byte pad: conflict-free)
            uint32_t* srow = reinterpret_cast<uint32_t*>(stg_q) + lane * rstride;
            const int buf = k & 1;
            role_wait(&a_full[buf], (uint32_t)(k >> 1) & 1u);
            if (et == 0) trace(p, TR_EPI_GO, k);
            tc_fence_after();
            for (int cc = c0; cc < bn; cc += cstep) {
                if (kDev && (p.exp & 4)) break;
                if (ob > 0 && (n0 + cc) / 32 >= Nw) break;  // past the last packed word (ragged last N tile)
                uint32_t acc[32];
                tmem_ld32(tmem_lane + (uint32_t)((buf * mt + sub) * bn) + cc, acc);
                tmem_wait_ld();
                if (p.pool_fused) {
                    // 2x2/2 max pooling on the codes (q is non-decreasing in v, reading R15):
                    // the window's pixels are lanes l, l^1, l^8, l^8^1 of this warp
                    uint32_t qb[8];
                    requant_chunk_bytes(acc, n0 + cc, cc, g, p.e, sTab, p.tab_mode, qb);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        qb[i] = __vmaxu4(qb[i], __shfl_xor_sync(0xffffffffu, qb[i], 1));
                        qb[i] = __vmaxu4(qb[i], __shfl_xor_sync(0xffffffffu, qb[i], 8));
                    }
                    if (valid && (tw & 1) == 0 && (hv & 1) == 0 && (n0 + cc) / 32 < Nw) {
                        uint32_t w[8];
                        bytes_to_words(qb, ob, w);
                        const long long prow = ((long long)b * p.Hp + (ho >> 1)) * p.Wp + (wo >> 1);
                        uint32_t* o = reinterpret_cast<uint32_t*>(p.Y) + prow * ob * Nw + (n0 + cc) / 32;
#pragma unroll
                        for (int tb = 0; tb < 8; tb++)
                            if (tb < ob) o[(long long)tb * Nw] = w[tb];
                    }
                } else if (ob == 0) {
                    stage_int32_chunk(acc, stg_w, lane);
                    __syncwarp();
                    const int j = lane & 7;
                    const int col = n0 + cc + 4 * j;
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int r = 4 * i + (lane >> 3);
                        const int mr = __shfl_sync(0xffffffffu, m, r);
                        const uint4 v = *reinterpret_cast<const uint4*>(stg_w + r * 128 + ((j ^ (r & 7)) << 4));
                        if (mr < g.M) {
                            int32_t* y = reinterpret_cast<int32_t*>(p.Y) + (long long)mr * g.N;
                            if ((g.N & 3) == 0 && col + 4 <= g.N) {
                                *reinterpret_cast<uint4*>(y + col) = v;
                            } else {
                                if (col < g.N) y[col] = (int32_t)v.x;
                                if (col + 1 < g.N) y[col + 1] = (int32_t)v.y;
                                if (col + 2 < g.N) y[col + 2] = (int32_t)v.z;
                                if (col + 3 < g.N) y[col + 3] = (int32_t)v.w;
                            }
                        }
                    }
                    __syncwarp();
                } else {
                    uint32_t w[8];
                    if (RES) {
                        uint32_t qb[8];
                        residual_chunk_bytes_tab(acc, m, n0 + cc, cc, g, p.e, sTab, qb);
                        bytes_to_words(qb, ob, w);
                    } else {
                        requant_chunk<false>(acc, n0 + cc, cc, g, p.e, sTab, p.tab_mode, w, m);
                    }
                    const int wi = cc >> 5;
#pragma unroll
                    for (int tb = 0; tb < 8; tb++)
                        if (tb < ob) srow[tb * nwt + wi] = w[tb];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(a_empty0 + 8u * (uint32_t)buf);
            if (et == 0) trace(p, TR_EPI_DONE, k);
            if (p.pool_fused) {
                if ((mt > 1 || half == 0) && n0 + bn >= g.N && valid && (tw & 1) == 0 && (hv & 1) == 0) {  // N padding
                    const long long prow = ((long long)b * p.Hp + (ho >> 1)) * p.Wp + (wo >> 1);
                    uint32_t* o = reinterpret_cast<uint32_t*>(p.Y) + prow * ob * Nw;
                    for (int tb = 0; tb < ob; tb++)
                        for (int wi = (n0 + bn) / 32; wi < Nw; wi++) o[(long long)tb * Nw + wi] = 0u;
                }
            } else if (ob > 0) {
                // padding words past the tile's columns (last N tile) are zero
                for (int wi = bn / 32 + (mt > 1 ? 0 : half); wi < nwt; wi += (mt > 1 ? 1 : 2))
                    for (int tb = 0; tb < ob; tb++) srow[tb * nwt + wi] = 0u;
                if (mt > 1) __syncwarp();
                else named_bar_sync(2 + qw, 64);  // both warps of the quarter staged their words
                if (m < g.M) {
                    uint32_t* orow = reinterpret_cast<uint32_t*>(p.Y) + (long long)m * ob * Nw + n0 / 32;
                    const int pw = nwt >> 2;  // 16-byte pieces per plane
                    for (int pc = (mt > 1 ? 0 : half); pc < ob * pw; pc += (mt > 1 ? 1 : 2)) {
                        const int tb = pw == 1 ? pc : pc >> 1, wq = pw == 1 ? 0 : (pc & 1) * 4;
                        *reinterpret_cast<uint4*>(orow + tb * Nw + wq) =
                            *reinterpret_cast<const uint4*>(srow + tb * nwt + wq);
                    }
                }
                if (mt > 1) __syncwarp();
                else named_bar_sync(2 + qw, 64);  // staging free for the next tile
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc2(tmem, p.tmem_cols);
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
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

// prepared int8 conv weights [C_out][R*S*Cp] bytes; box {128 bytes = one (tap, channel block)
// k-block, rows} landing in the UMMA K-major SWIZZLE_128B layout
static bool make_w_map(CUtensorMap* m, const uint8_t* base, int N, int Kp, int rows) {
    PFN_encodeTiled enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)Kp};
    cuuint32_t box[2] = {128, (cuuint32_t)rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr size_t kSmemMax = 227 * 1024;

// Fill the tiling / buffering plan; false when the shape does not fit this kernel.
static bool plan(const Geom& g, const Epi& e, Params& p, int sms = 148) {
    std::memset(&p, 0, sizeof(p));
    p.g = g;
    p.e = e;
    if (!g.conv || g.M <= 0 || g.N <= 0 || g.K <= 0 || g.RS > 60) return false;  // tap table: 60 entries
    const int R = g.RS / g.S;
    p.B = g.M / (g.Ho * g.Wo);
    p.E = (R - 1) / g.stride;
    p.Hv = g.Ho + p.E;
    if (e.pool && (p.Hv & 1)) p.Hv++;  // pooled windows must start on even tall rows (one more separator)
    p.nrho = g.stride < R ? g.stride : R;
    p.ncopy = p.nrho * g.S;
    p.mt = 1;
    p.th = TH;
    p.stg = STG1;
    p.crow = TH + p.E;
    p.cl = g.C > 64 ? 128 : (g.C > 32 ? 64 : 32);
    p.cc8 = p.cl * 8;
    p.smask = p.cl / 16 - 1;
    p.G = ((g.C < 128 ? g.C : 128) + 31) / 32;
    p.nchunk = g.CB;
    p.ixn = g.stride * (TW - 1) + g.S;
    if (p.G * p.ixn > DEC_THREADS || (g.S + g.stride - 1) / g.stride > kMaxTg) return false;  // decode split / targets
    p.copy_bytes = (uint32_t)(p.crow * p.cc8);
    p.set_bytes = (uint32_t)p.ncopy * p.copy_bytes;
    p.nsteps = g.RS * p.nchunk;
    p.bn = g.N > 128 ? 256 : (g.N > 64 ? 128 : 64);
    p.tiles_c = (g.Wo + TW - 1) / TW;
    const long long rows_tiles = ((long long)p.B * p.Hv + TH - 1) / TH;
    const long long cta_tiles = rows_tiles * p.tiles_c;
    if (cta_tiles > (1LL << 30) || (long long)p.B * p.Hv > (1LL << 30)) return false;
    p.cta_tiles = (int)cta_tiles;
    p.pair_tiles = (p.cta_tiles + 1) / 2;
    // narrower N tiles while fewer than half the CTA pairs would get a tile (measured on the C3
    // layers at batch 64: 7x7 and 14x14 stride-2 maps run 10 % faster at bn = 128)
    // (packed outputs keep whole 128-column words groups per tile: bn >= 128 unless N <= 64)
    const int bn_min = (e.out_bits > 0 && g.N > 64) ? 128 : 64;
    while (p.bn > bn_min && (long long)p.pair_tiles * ((g.N + p.bn - 1) / p.bn) < sms / 4) p.bn /= 2;
#if APNN_DEV
    {
        const char* b = getenv("APNN_HALO_BN");
        if (b && atoi(b) >= 64 && atoi(b) <= 256) p.bn = atoi(b);
    }
#endif
    p.n_tiles = (g.N + p.bn - 1) / p.bn;
    p.num_tiles = p.pair_tiles * p.n_tiles;
    // two 128-row sub-tiles per CTA tile (32 tall rows) when the N tile leaves TMEM room for two
    // double-buffered accumulators and every pair still gets >= 2 tiles: the per-tile hand-offs
    // and the MMA issuer's per-tap work are paid once per 256 rows
    {
        const long long rt2 = ((long long)p.B * p.Hv + 2 * TH - 1) / (2 * TH);
        const long long pt2 = (rt2 * p.tiles_c + 1) / 2;
        const size_t set2 = (size_t)p.ncopy * (2 * TH + p.E) * p.cc8;
        const size_t fixed2 = EPI_WARPS * (size_t)STG2 + (size_t)p.bn * kTabStride * 4 + (3 * MAX_WS + 8) * 8 +
                              16 + 4 * 64 + 256 + 1024;
        bool two = p.bn <= 128 && pt2 * p.n_tiles >= 2LL * (sms / 2) &&
                   fixed2 + 2 * set2 + 4 * (size_t)(p.bn / 2) * 128 <= kSmemMax;
#if APNN_DEV
        if (getenv("APNN_HALO_MT"))
            two = atoi(getenv("APNN_HALO_MT")) == 2 && p.bn <= 128 && fixed2 + 2 * set2 + 4 * (size_t)(p.bn / 2) * 128 <= kSmemMax;
#endif
        if (two) {
            p.mt = 2;
            p.stg = STG2;
            p.th = 2 * TH;
            p.crow = p.th + p.E;
            p.copy_bytes = (uint32_t)(p.crow * p.cc8);
            p.set_bytes = (uint32_t)p.ncopy * p.copy_bytes;
            p.cta_tiles = (int)(rt2 * p.tiles_c);
            p.pair_tiles = (p.cta_tiles + 1) / 2;
            p.num_tiles = p.pair_tiles * p.n_tiles;
        }
    }
    // epilogue: 2x2/2 max pooling of whole windows (tile rows/cols even, images start on even rows)
    if (e.pool) {
        if (!(e.pool == 2 && e.pool_stride == 2 && !e.pool_avg && e.out_bits > 0 && g.Ho % 2 == 0 &&
              g.Wo % 2 == 0 && p.Hv % 2 == 0))
            return false;
        p.pool_fused = 1;
        p.Hp = g.Ho / 2;
        p.Wp = g.Wo / 2;
    }
    p.tab_mode = kTabNone;
    if (e.res) p.tab_mode = kTabResidual;
    else if (e.out_bits > 0 && e.out_bits <= 2) p.tab_mode = kTabQ3;
    else if (e.out_bits > 2 && (unsigned long long)e.qmax * (unsigned long long)e.S <= 0xFFFFFFFFull)
        p.tab_mode = kTabHybrid;
    // shared memory: weights + copies + store staging + table + barriers
    const size_t wstage = (size_t)(p.bn / 2) * 128;
    const size_t fixed = EPI_WARPS * (size_t)p.stg + (size_t)p.bn * kTabStride * 4 + (3 * MAX_WS + 8) * 8 + 16 + 4 * 64 + 256 + 1024;
    if (fixed + p.set_bytes + 2 * wstage > kSmemMax) return false;
    const size_t budget = kSmemMax - fixed;
    if (p.n_tiles == 1 && p.nsteps <= MAX_WS && (size_t)p.nsteps * wstage + 2 * (size_t)p.set_bytes <= budget) {
        p.w_resident = 1;
        p.ws = p.nsteps;
        p.nbuf = 2;
    } else {
        p.nbuf = (2 * (size_t)p.set_bytes + 4 * wstage <= budget) ? 2 : 1;
        size_t ws = (budget - p.nbuf * (size_t)p.set_bytes) / wstage;
        if (ws > MAX_WS) ws = MAX_WS;
        if (ws < 2) return false;
        p.ws = (int)ws;
    }
    {
        uint32_t cols = 32;
        while (cols < (uint32_t)(2 * p.mt * p.bn)) cols <<= 1;
        p.tmem_cols = cols;
    }
    return true;
}

static size_t smem_bytes(const Params& p) {
    return (size_t)p.ws * (p.bn / 2) * 128 + (size_t)p.nbuf * p.set_bytes + EPI_WARPS * (size_t)p.stg +
           (size_t)p.bn * kTabStride * 4 + (3 * MAX_WS + 8) * 8 + 16 + 4 * 64 + 256;
}

template <bool AP, bool WP, bool RES, bool RAW = false>
static cudaError_t launch(const CUtensorMap& tw, const Params& p, int grid, size_t smem, cudaStream_t s) {
    auto kfn = halo_kernel<AP, WP, RES, RAW>;
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
    if (err != cudaSuccess) return err;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // the kernel waits (griddepcontrol)
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    err = cudaLaunchKernelEx(&cfg, kfn, tw, p);
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

}  // namespace halo

// Can the tap-reuse kernel run this prepared-weight convolution?
bool conv_halo_supports(const Geom& g, const Epi& e) {
    halo::Params p;
    return halo::plan(g, e, p);
}

cudaError_t launch_conv_halo(const uint32_t* X, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y, int sms,
                             cudaStream_t s) {
    using namespace halo;
    Params p;
    if (!plan(g, e, p, sms)) return cudaErrorNotSupported;
    p.X = X;
    p.Y = Y;
#if APNN_DEV
    p.exp = getenv("APNN_HALO_EXP") ? atoi(getenv("APNN_HALO_EXP")) : 0;
    const char* trace_path = getenv("APNN_HALO_TRACE");
    const size_t tr_bytes = sizeof(unsigned long long) * 2 * TR_NEV * kTrN;
    if (trace_path) {  // development only: allocates and synchronises
        cudaMalloc(&p.trace, tr_bytes);
        cudaMemset(p.trace, 0, tr_bytes);
    }
#endif
    CUtensorMap tw;
    if (!make_w_map(&tw, Wp, g.N, g.RS * g.Cw * 32, p.bn / 2)) return cudaErrorInvalidValue;
    int pairs = sms / 2;
    if (pairs > p.num_tiles) pairs = p.num_tiles;
    if (pairs < 1) pairs = 1;
    const size_t smem = smem_bytes(p) + 1024;
    const bool apm = g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_01_A_PM1;
    const bool wpm = g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_PM1_A_01;
    cudaError_t err;
    if (e.res) {
        if (apm) return cudaErrorNotSupported;
        err = wpm ? launch<false, true, true>(tw, p, 2 * pairs, smem, s) : launch<false, false, true>(tw, p, 2 * pairs, smem, s);
    } else if (apm) {
        err = wpm ? launch<true, true, false>(tw, p, 2 * pairs, smem, s) : launch<true, false, false>(tw, p, 2 * pairs, smem, s);
    } else {
        err = wpm ? launch<false, true, false>(tw, p, 2 * pairs, smem, s) : launch<false, false, false>(tw, p, 2 * pairs, smem, s);
    }
    count_launch();
#if APNN_DEV
    if (p.trace) {
        cudaStreamSynchronize(s);
        unsigned long long* h = (unsigned long long*)malloc(tr_bytes);
        cudaMemcpy(h, p.trace, tr_bytes, cudaMemcpyDeviceToHost);
        FILE* f = fopen(trace_path, "wb");
        if (f) { fwrite(h, 1, tr_bytes, f); fclose(f); }
        free(h);
        cudaFree(p.trace);
    }
#endif
    return err;
}

// The first layer on the tap-reuse kernel (raw mode): X is the raw 8-bit NHWC image [B][H][W][C],
// Wp the prepared weights of W viewed as C_out*R rows of S*C_in (window order (s, c)).
bool conv_first_supports(const Geom& g0, const Epi& e, int S_raw, int C_raw) {
    Geom g = g0;
    halo::Params p;
    if (S_raw * C_raw > 128 || g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_01_A_PM1 || e.res) return false;
    return halo::plan(g, e, p);
}

cudaError_t launch_conv_first(const uint8_t* X, const uint8_t* Wp, const Geom& g, const Epi& e, int qz, int qs,
                              int S_raw, int C_raw, void* Y, int sms, cudaStream_t s) {
    using namespace halo;
    Params p;
    if (!conv_first_supports(g, e, S_raw, C_raw) || !plan(g, e, p, sms)) return cudaErrorNotSupported;
    p.Xraw = X;
    p.Y = Y;
    p.raw = 1;
    p.qz = qz;
    p.qs = qs;
    p.S_raw = S_raw;
    p.C_raw = C_raw;
#if APNN_DEV
    p.exp = getenv("APNN_HALO_EXP") ? atoi(getenv("APNN_HALO_EXP")) : 0;
    const char* trace_path = getenv("APNN_HALO_TRACE");
    const size_t tr_bytes = sizeof(unsigned long long) * 2 * TR_NEV * kTrN;
    if (trace_path) {
        cudaMalloc(&p.trace, tr_bytes);
        cudaMemset(p.trace, 0, tr_bytes);
    }
#endif
    CUtensorMap tw;
    if (!make_w_map(&tw, Wp, g.N, g.RS * 128, p.bn / 2)) return cudaErrorInvalidValue;  // rows of R x 128 B
    int pairs = sms / 2;
    if (pairs > p.num_tiles) pairs = p.num_tiles;
    if (pairs < 1) pairs = 1;
    const size_t smem = smem_bytes(p) + 1024;
    const bool wpm = g.enc == APNN_ENC_W_PM1_A_01;
    cudaError_t err = wpm ? launch<false, true, false, true>(tw, p, 2 * pairs, smem, s)
                          : launch<false, false, false, true>(tw, p, 2 * pairs, smem, s);
    count_launch();
#if APNN_DEV
    if (p.trace) {
        cudaStreamSynchronize(s);
        unsigned long long* h = (unsigned long long*)malloc(tr_bytes);
        cudaMemcpy(h, p.trace, tr_bytes, cudaMemcpyDeviceToHost);
        FILE* f = fopen(trace_path, "wb");
        if (f) { fwrite(h, 1, tr_bytes, f); fclose(f); }
        free(h);
        cudaFree(p.trace);
    }
#endif
    return err;
}

}  // namespace apnn
