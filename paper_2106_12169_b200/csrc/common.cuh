// common.cuh -- shared device/host helpers of libapnn (B200, sm_100a).
//
// Operand addressing for the AP-bit contraction.  GEMM and convolution are the
// same loop (APConv as implicit GEMM): the reduction runs
// over "chunks" of 128 elements; chunk kc of the reduction is
//     rs = kc / CB (filter tap, r*S+s),  cb = kc % CB (128-channel block)
// and for a GEMM RS = 1, CB = Kw/4.  A chunk of any packed row is 4 uint32 words
// per plane at  base + (row * bits + t) * Cw + cb * 4  (include/apnn.h layout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/apnn.h"

namespace apnn {

// -------------------------------------------------------------- host side
void count_launch(int n = 1);  // apnn_launch_count bookkeeping (apnn.cu)

// Geometry of one contraction: everything a kernel needs to turn (row, chunk)
// into addresses.  Passed by value as a kernel parameter.
struct Geom {
    int M, N;          // output rows (GEMM M or B*Ho*Wo) and columns (N or C_out)
    int K;             // logical reduction length (GEMM K; conv R*S*C_in)
    int a_bits, w_bits;
    int enc;           // apnn_encoding
    int nchunks;       // number of 128-element chunks in the reduction
    int Cw;            // words per plane run of one packed row (GEMM: Kw; conv: Cp/32)
    int CB;            // 128-element blocks per plane run (Cw / 4)
    int C;             // logical elements per plane run (GEMM: K; conv: C_in)
    int RS;            // filter taps (GEMM: 1)
    // conv geometry (unused for GEMM)
    int conv;
    int H, W, Ho, Wo, S, stride, pad;
};

// Tile configuration of the int8 tensor-core kernels (row f4, tuner.cu): kernel 1 = one-CTA
// 128 x bn tile with a split-K cluster of z CTAs, kernel 2 = CTA pair 256 x bn.
struct TileCfg {
    int kernel, bm, bn, z;
    long long tlp;  // CTAs launched (the paper's TLP, Eq. TLP adapted)
    double ci;      // Eq. CI of the tile
};
TileCfg tune_tiles(int M, int N, int K, int T, bool packed);
bool tile_cfg_valid(const TileCfg& c, int M, int N, int K, bool packed);

// Per-row context for gathering A chunks (computed once per row per tile).
struct RowCtx {
    long long pix;  // GEMM: m; conv: b*H*W (base pixel index of image b)
    int hb, wb;     // conv: ho*stride - pad, wo*stride - pad
    bool valid;     // m < M
};

__device__ __forceinline__ RowCtx make_row(const Geom& g, int m) {
    RowCtx c;
    c.valid = m < g.M;
    if (!g.conv) {
        c.pix = m;
        c.hb = c.wb = 0;
    } else {
        int mm = c.valid ? m : 0;
        int hw = g.Ho * g.Wo;
        int b = mm / hw;
        int rem = mm - b * hw;
        int ho = rem / g.Wo;
        int wo = rem - ho * g.Wo;
        c.pix = (long long)b * g.H * g.W;
        c.hb = ho * g.stride - g.pad;
        c.wb = wo * g.stride - g.pad;
    }
    return c;
}

// Address of plane 0 of chunk kc of A row `c`, or nullptr if the chunk is
// out of frame (value 0) or the row is beyond M.
// *nvalid = number of logical (non-padding) elements in the chunk.
__device__ __forceinline__ const uint32_t* a_chunk(const uint32_t* A, const Geom& g,
                                                   const RowCtx& c, int kc, int* nvalid) {
    if (!c.valid) { *nvalid = 0; return nullptr; }
    int rs = 0, cb = kc;
    long long pix = c.pix;
    if (g.conv) {
        rs = kc / g.CB;
        cb = kc - rs * g.CB;
        int r = rs / g.S, s = rs - (rs / g.S) * g.S;
        int hi = c.hb + r, wi = c.wb + s;
        if (hi < 0 || hi >= g.H || wi < 0 || wi >= g.W) { *nvalid = 0; return nullptr; }
        pix += (long long)hi * g.W + wi;
    }
    int rem = g.C - cb * 128;
    *nvalid = rem < 128 ? rem : 128;
    return A + (pix * g.a_bits) * g.Cw + cb * 4;
}

// Address of plane 0 of chunk kc of weight row n (n < N assumed).
__device__ __forceinline__ const uint32_t* b_chunk(const uint32_t* W, const Geom& g, int n, int kc) {
    int rs = 0, cb = kc;
    if (g.conv) { rs = kc / g.CB; cb = kc - rs * g.CB; }
    return W + ((long long)(n * g.RS + rs) * g.w_bits) * g.Cw + cb * 4;
}

// ---------------------------------------------------------------- epilogue
// The fused element-wise routine, integer form:
//   v = alpha*y + beta (int64);  q = clamp(floor(v / S), 0, qmax)
struct Epi {
    const int32_t* alpha;  // may be nullptr (= 1)
    const int32_t* beta;   // may be nullptr (= 0)
    int32_t S;
    int32_t out_bits;      // 0 -> raw int32 output
    int32_t qmax;
    float invS;            // 1/S (rounded), used for a first guess only
    int32_t pool;          // conv pooling window k (0 = none)
    int32_t pool_stride;
    int32_t pool_avg;      // 0 max, 1 average
    const void* res;       // residual shortcut z (reading R24) or nullptr: int32 [M][N] (res_bits 0)
    int32_t res_bits;      //   or packed codes [M][res_bits][Nw]
    const int32_t* rho;    // per-column residual scale or nullptr (= 1)
};

// q = clamp(floor(v / S), 0, qmax) for an int64 v (the quantisation step alone)
__device__ __forceinline__ uint32_t quantise_v(const Epi& e, long long v) {
    if (v < 0) return 0;
    long long lim = (long long)(e.qmax + 1) * e.S;
    if (v >= lim) return (uint32_t)e.qmax;
    int q = __float2int_rz((float)v * e.invS);
    long long r = v - (long long)q * e.S;
    while (r < 0) { q -= 1; r += e.S; }
    while (r >= e.S) { q += 1; r -= e.S; }
    return (uint32_t)q;
}

__device__ __forceinline__ uint32_t requant(const Epi& e, int32_t y, int32_t alpha, int32_t beta) {
    long long v = (long long)alpha * y + beta;
    if (v < 0) return 0;
    long long lim = (long long)(e.qmax + 1) * e.S;
    if (v >= lim) return (uint32_t)e.qmax;
    // 0 <= v < 256*S: first guess in fp32, then exact integer correction.
    int q = __float2int_rz((float)v * e.invS);
    long long r = v - (long long)q * e.S;
    while (r < 0) { q -= 1; r += e.S; }
    while (r >= e.S) { q += 1; r -= e.S; }
    return (uint32_t)q;
}

__device__ __forceinline__ int32_t epi_alpha(const Epi& e, int n) { return e.alpha ? __ldg(e.alpha + n) : 1; }
__device__ __forceinline__ int32_t epi_beta(const Epi& e, int n) { return e.beta ? __ldg(e.beta + n) : 0; }

// Bit t of each byte of `u` gathered into a nibble (bit i of result = bit t of byte i).
__device__ __forceinline__ uint32_t byte_bits_to_nibble(uint32_t u, int t) {
    uint32_t x = (u >> t) & 0x01010101u;
    return ((x * 0x00204081u) >> 21) & 0xFu;  // shifted copies land on bits 21..24 without carries
}

}  // namespace apnn
