/*
 * apnn_oracle.c -- CPU oracle for the APNN-TC hot path (arXiv 2106.12169).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the slow, obviously-correct
 * reference the CUDA path is checked against.  Only tests/, the smoke() entry
 * point and bench.py's cpu_baseline / --impl reference legs may load it.  It
 * shares no code, header, table or constant with the product library
 * (paper_2106_12169_b200/csrc, include/apnn.h) and neither side includes the
 * other.
 *
 * Everything here is integer arithmetic, so "fp64 by default" does not apply:
 * accumulation is int64 and every result is checked to fit in int32
 * ("APMM generates 32-bit output to avoid data overflow").
 *
 * Conventions:
 *   A  = activations (features), M x K unsigned codes, one byte per code.
 *   W  = weights, N x K unsigned codes, one byte per code.
 *   Y  = A . W^T, M x N int32.
 *   The paper writes W^(s) M x K and X^(t) N x K; we name the
 *   operands by role instead (reading R4).
 *   encoding (reading R5/R6):
 *     0  A 0/1 codes, W 0/1 codes                (Case I,  AND + popc)
 *     1  A +-1,       W +-1,  a_bits = w_bits = 1 (Case II, XOR + popc)
 *     2  A 0/1 codes, W +-1,  w_bits = 1          (Case III, linear transform + AND)
 *     3  A +-1,       W 0/1,  a_bits = 1          (Case III with roles swapped)
 *   A +-1 operand stores -1 as bit 0 and +1 as bit 1 (PAPER.md:1456,
 *   "we first map -1 to 0").
 *
 * Functions:
 *   oracle_gemm           plain definition  Y[m][n] = sum_k dec(A[m][k]) dec(W[n][k])
 *   oracle_gemm_bitplane  the paper's AP-bit method, step by step:
 *                           bit decomposition  (Eq. bitDecomposition)
 *                           1-bit products with data-adaptive operator selection
 *                                              (Cases I-III)
 *                           bit combination
 *   oracle_conv2d         plain direct convolution, value-domain zero padding
 *                           (APConv PAPER.md:1612-1613, input-aware padding 1652-1662)
 *   oracle_epilogue       fused requantisation  q = clamp(floor((alpha*y + beta)/S), 0, 2^b-1)
 *                           (quantisation PAPER.md:1283-1287, fused formula 1303-1306)
 *   oracle_pool_epilogue  BN affine -> k x k pooling (max or average) -> quantisation
 *                           (pooling PAPER.md:1293, fused conv+pool+quant 641-647,
 *                            layer order of the fused formula 1299-1306; reading R15)
 *   oracle_pack           byte-exact packed bit-plane format [rows][bits][Kp/32]
 *                           (decomposition PAPER.md:1419-1421, packing 1255-1256)
 *
 * Parity pins for every function live in tests/test_oracle.py (numpy/torch
 * library routines, brute force, the paper's worked examples).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_BITS 1
#define OR_ERR_ENC 2
#define OR_ERR_CODE 3
#define OR_ERR_OVERFLOW 4
#define OR_ERR_SHAPE 5

/* ---------------------------------------------------------------- helpers */

/* which operands are +-1 encoded, and is the (enc, bits) pair legal */
static int enc_check(int enc, int a_bits, int w_bits, int *a_pm1, int *w_pm1)
{
    if (a_bits < 1 || a_bits > 8 || w_bits < 1 || w_bits > 8) return OR_ERR_BITS;
    switch (enc) {
    case 0: *a_pm1 = 0; *w_pm1 = 0; return OR_OK;
    case 1: *a_pm1 = 1; *w_pm1 = 1; return (a_bits == 1 && w_bits == 1) ? OR_OK : OR_ERR_ENC;
    case 2: *a_pm1 = 0; *w_pm1 = 1; return (w_bits == 1) ? OR_OK : OR_ERR_ENC;
    case 3: *a_pm1 = 1; *w_pm1 = 0; return (a_bits == 1) ? OR_OK : OR_ERR_ENC;
    default: return OR_ERR_ENC;
    }
}

/* value of a stored code: 0/1 encoding -> the code itself; +-1 -> 2u-1
 * (bit 0 means -1, bit 1 means +1) */
static int64_t dec(unsigned u, int pm1) { return pm1 ? 2 * (int64_t)u - 1 : (int64_t)u; }

static int codes_in_range(const uint8_t *x, size_t n, int bits)
{
    for (size_t i = 0; i < n; i++)
        if (x[i] >> bits) return 0;
    return 1;
}

static int fits_i32(int64_t v) { return v >= INT32_MIN && v <= INT32_MAX; }

static void set_threads(int threads)
{
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------- plain definition */

/* Y[m][n] = sum_k dec(A[m][k]) * dec(W[n][k]), int64 accumulate, int32 result.
 * This is the definition the AP-bit method must reproduce (PAPER.md:1410,
 * "We note that Y = WX mathematically"). */
int oracle_gemm(const uint8_t *A, const uint8_t *W, int M, int N, int K,
                int a_bits, int w_bits, int enc, int32_t *Y, int threads)
{
    int a_pm1, w_pm1;
    int st = enc_check(enc, a_bits, w_bits, &a_pm1, &w_pm1);
    if (st) return st;
    if (M < 0 || N < 0 || K < 0) return OR_ERR_SHAPE;
    if (!codes_in_range(A, (size_t)M * K, a_bits) || !codes_in_range(W, (size_t)N * K, w_bits))
        return OR_ERR_CODE;
    set_threads(threads);
    int overflow = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : overflow)
    for (int m = 0; m < M; m++) {
        for (int n = 0; n < N; n++) {
            int64_t acc = 0;
            for (int k = 0; k < K; k++)
                acc += dec(A[(size_t)m * K + k], a_pm1) * dec(W[(size_t)n * K + k], w_pm1);
            if (!fits_i32(acc)) overflow = 1;
            Y[(size_t)m * N + n] = (int32_t)acc;
        }
    }
    return overflow ? OR_ERR_OVERFLOW : OR_OK;
}

/* ------------------------------------------------ the paper's AP-bit method */

/* Eq. bitDecomposition: plane t of row r is
 * (x >> t) & 1, packed LSB-first into 64-bit words of ceil(K/64) per row.
 * Returns a malloc'ed array [rows][bits][KW]. */
static uint64_t *decompose64(const uint8_t *x, int rows, int K, int bits, int KW)
{
    uint64_t *p = (uint64_t *)calloc((size_t)rows * bits * KW + 1, sizeof(uint64_t));
    for (int r = 0; r < rows; r++)
        for (int t = 0; t < bits; t++)
            for (int k = 0; k < K; k++)
                if ((x[(size_t)r * K + k] >> t) & 1)
                    p[((size_t)r * bits + t) * KW + k / 64] |= (uint64_t)1 << (k % 64);
    return p;
}

static int64_t popc_and(const uint64_t *a, const uint64_t *b, int KW)
{
    int64_t c = 0;
    for (int i = 0; i < KW; i++) c += __builtin_popcountll(a[i] & b[i]);
    return c;
}
static int64_t popc_xor(const uint64_t *a, const uint64_t *b, int KW)
{
    int64_t c = 0;
    for (int i = 0; i < KW; i++) c += __builtin_popcountll(a[i] ^ b[i]);
    return c;
}
static int64_t popc1(const uint64_t *a, int KW)
{
    int64_t c = 0;
    for (int i = 0; i < KW; i++) c += __builtin_popcountll(a[i]);
    return c;
}

/* The AP-bit operation template with data-adaptive
 * operator selection:
 *   1. decompose A into a_bits planes X^(t) and W into w_bits planes W^(s);
 *   2. for every (s, t) compute the 1-bit product Y^(s,t) with the operator the
 *      encodings select:
 *        Case I   (0/1 x 0/1):  popc(W AND X)
 *        Case II  (+-1 x +-1):  n - 2 popc(W XOR X), n = logical K
 *        Case III (+-1 W, 0/1 X): W^ = (W + J)/2 is the stored bit;
 *                               WX = 2 popc(W^ AND X) - J.X,  J.X = popc(X)
 *        (encoding 3 is Case III with the roles of W and X swapped)
 *   3. bit combination  Y = sum_s sum_t 2^(s+t) Y^(s,t)
 * Padding bits of the last word are zero in both operands, so they add
 * nothing to AND/XOR popcounts; Case II uses the logical length K for n. */
int oracle_gemm_bitplane(const uint8_t *A, const uint8_t *W, int M, int N, int K,
                         int a_bits, int w_bits, int enc, int32_t *Y, int threads)
{
    int a_pm1, w_pm1;
    int st = enc_check(enc, a_bits, w_bits, &a_pm1, &w_pm1);
    if (st) return st;
    if (M < 0 || N < 0 || K < 0) return OR_ERR_SHAPE;
    if (!codes_in_range(A, (size_t)M * K, a_bits) || !codes_in_range(W, (size_t)N * K, w_bits))
        return OR_ERR_CODE;
    int KW = (K + 63) / 64;
    uint64_t *X = decompose64(A, M, K, a_bits, KW); /* X^(t): [M][a_bits][KW] */
    uint64_t *Wp = decompose64(W, N, K, w_bits, KW); /* W^(s): [N][w_bits][KW] */
    set_threads(threads);
    int overflow = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : overflow)
    for (int m = 0; m < M; m++) {
        for (int n = 0; n < N; n++) {
            int64_t y = 0;
            for (int s = 0; s < w_bits; s++) {
                for (int t = 0; t < a_bits; t++) {
                    const uint64_t *xt = X + ((size_t)m * a_bits + t) * KW;
                    const uint64_t *ws = Wp + ((size_t)n * w_bits + s) * KW;
                    int64_t yst;
                    if (!a_pm1 && !w_pm1)       /* Case I */
                        yst = popc_and(ws, xt, KW);
                    else if (a_pm1 && w_pm1)    /* Case II */
                        yst = (int64_t)K - 2 * popc_xor(ws, xt, KW);
                    else if (w_pm1)             /* Case III: W +-1, X 0/1 */
                        yst = 2 * popc_and(ws, xt, KW) - popc1(xt, KW);
                    else                        /* Case III, roles swapped: X +-1, W 0/1 */
                        yst = 2 * popc_and(xt, ws, KW) - popc1(ws, KW);
                    y += yst * ((int64_t)1 << (s + t)); /* bit combination */
                }
            }
            if (!fits_i32(y)) overflow = 1;
            Y[(size_t)m * N + n] = (int32_t)y;
        }
    }
    free(X);
    free(Wp);
    return overflow ? OR_ERR_OVERFLOW : OR_OK;
}

/* --------------------------------------------------------------- APConv */

/* Direct convolution over unpacked codes (APConv):
 *   X  NHWC codes [B][H][W][C],  Wt  OHWI codes [Co][R][S][C]
 *   Y[b][ho][wo][co] = sum_{r,s,c} dec(X[b][ho*st+r-pad][wo*st+s-pad][c]) * dec(Wt[co][r][s][c])
 * Taps that fall outside the frame contribute the VALUE 0 for every
 * encoding.  This is the semantics the paper's input-aware padding
 * implements: pad 0 for 0/1 features, and for +-1
 * features pad 1 and subtract the out-of-frame count (reading R16).
 *   Ho = floor((H + 2 pad - R)/st) + 1, likewise Wo. */
int oracle_conv2d(const uint8_t *X, const uint8_t *Wt, int B, int H, int Wd, int C, int Co,
                  int R, int S, int stride, int pad, int a_bits, int w_bits, int enc,
                  int32_t *Y, int threads)
{
    int a_pm1, w_pm1;
    int st = enc_check(enc, a_bits, w_bits, &a_pm1, &w_pm1);
    if (st) return st;
    if (B < 0 || H < 1 || Wd < 1 || C < 1 || Co < 1 || R < 1 || S < 1 || stride < 1 || pad < 0)
        return OR_ERR_SHAPE;
    int Ho = (H + 2 * pad - R) / stride + 1;
    int Wo = (Wd + 2 * pad - S) / stride + 1;
    if (Ho < 1 || Wo < 1) return OR_ERR_SHAPE;
    if (!codes_in_range(X, (size_t)B * H * Wd * C, a_bits) ||
        !codes_in_range(Wt, (size_t)Co * R * S * C, w_bits))
        return OR_ERR_CODE;
    set_threads(threads);
    int overflow = 0;
    long long npix = (long long)B * Ho * Wo;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : overflow)
    for (long long p = 0; p < npix; p++) {
        int b = (int)(p / ((long long)Ho * Wo));
        int ho = (int)((p / Wo) % Ho);
        int wo = (int)(p % Wo);
        for (int co = 0; co < Co; co++) {
            int64_t acc = 0;
            for (int r = 0; r < R; r++) {
                int hi = ho * stride + r - pad;
                if (hi < 0 || hi >= H) continue;           /* out of frame: value 0 */
                for (int s = 0; s < S; s++) {
                    int wi = wo * stride + s - pad;
                    if (wi < 0 || wi >= Wd) continue;      /* out of frame: value 0 */
                    const uint8_t *xp = X + (((size_t)b * H + hi) * Wd + wi) * C;
                    const uint8_t *wp = Wt + (((size_t)co * R + r) * S + s) * C;
                    for (int c = 0; c < C; c++) acc += dec(xp[c], a_pm1) * dec(wp[c], w_pm1);
                }
            }
            if (!fits_i32(acc)) overflow = 1;
            Y[(size_t)p * Co + co] = (int32_t)acc;
        }
    }
    return overflow ? OR_ERR_OVERFLOW : OR_OK;
}

/* ------------------------------------------------------------- epilogue */

/* floor(v / d) for d > 0, rounding toward minus infinity (reading R11). */
static int64_t floor_div(int64_t v, int64_t d)
{
    int64_t q = v / d;             /* C truncates toward zero */
    if (v % d != 0 && v < 0) q -= 1;
    return q;
}

/* Fused requantisation (semantic-aware kernel fusion):
 *   v = alpha[n] * Y[m][n] + beta[n]          (int64; BN / zero point folded
 *                                              on the host into integers, R12)
 *   q = clamp(floor(v / S), 0, 2^out_bits - 1) (quantisation PAPER.md:1285;
 *                                              ReLU = the lower clamp, R14)
 * alpha == NULL means 1, beta == NULL means 0.  Writes one code per byte. */
int oracle_epilogue(const int32_t *Y, int M, int N, const int32_t *alpha, const int32_t *beta,
                    int32_t S, int out_bits, uint8_t *q)
{
    if (out_bits < 1 || out_bits > 8) return OR_ERR_BITS;
    if (S <= 0 || M < 0 || N < 0) return OR_ERR_SHAPE;
    int64_t qmax = ((int64_t)1 << out_bits) - 1;
    for (int m = 0; m < M; m++) {
        for (int n = 0; n < N; n++) {
            int64_t a = alpha ? alpha[n] : 1;
            int64_t b = beta ? beta[n] : 0;
            int64_t v = a * (int64_t)Y[(size_t)m * N + n] + b;
            int64_t f = floor_div(v, S);
            if (f < 0) f = 0;
            if (f > qmax) f = qmax;
            q[(size_t)m * N + n] = (uint8_t)f;
        }
    }
    return OR_OK;
}

/* Pooling between the BN affine and the quantisation (reading R15; pooling
 * PAPER.md:1293 "splits the feature map spatially into k x k grids and generates
 * 1 scalar output for each grid by computing the average or the maximum value";
 * fused conv + pooling + quantisation PAPER.md:641-647):
 *   v[b][h][w][n] = alpha[n] * Y[b][h][w][n] + beta[n]                 (int64)
 *   P[b][i][j][n] = max over the k x k grid at (i*st, j*st) of v        (avg = 0), or
 *                 = floor( sum over the grid of v / k^2 )               (avg = 1)
 *   q = clamp(floor(P / S), 0, 2^out_bits - 1)
 * Y is NHWC int32 [B][H][W][N]; q is [B][Hp][Wp][N] codes, Hp = (H - k)/st + 1
 * (grids that do not fit are dropped, "floor" pooling). */
int oracle_pool_epilogue(const int32_t *Y, int B, int H, int Wd, int N, const int32_t *alpha,
                         const int32_t *beta, int32_t S, int out_bits, int k, int stride, int avg,
                         uint8_t *q)
{
    if (out_bits < 1 || out_bits > 8) return OR_ERR_BITS;
    if (S <= 0 || B < 0 || H < 1 || Wd < 1 || N < 0 || k < 1 || stride < 1 || k > H || k > Wd)
        return OR_ERR_SHAPE;
    int Hp = (H - k) / stride + 1, Wp = (Wd - k) / stride + 1;
    int64_t qmax = ((int64_t)1 << out_bits) - 1;
    for (int b = 0; b < B; b++)
        for (int i = 0; i < Hp; i++)
            for (int j = 0; j < Wp; j++)
                for (int n = 0; n < N; n++) {
                    int64_t a = alpha ? alpha[n] : 1;
                    int64_t c = beta ? beta[n] : 0;
                    int64_t best = 0, sum = 0;
                    for (int r = 0; r < k; r++)
                        for (int s = 0; s < k; s++) {
                            int h = i * stride + r, w = j * stride + s;
                            int64_t v = a * (int64_t)Y[(((size_t)b * H + h) * Wd + w) * N + n] + c;
                            if ((r == 0 && s == 0) || v > best) best = v;
                            sum += v;
                        }
                    int64_t P = avg ? floor_div(sum, (int64_t)k * k) : best;
                    int64_t f = floor_div(P, S);
                    if (f < 0) f = 0;
                    if (f > qmax) f = qmax;
                    q[(((size_t)b * Hp + i) * Wp + j) * N + n] = (uint8_t)f;
                }
    return OR_OK;
}

/* ---------------------------------------------------------------- packing */

/* Packed bit-plane format (the library contract):
 *   out[(r * bits + t) * Kw + k / 32] bit (k % 32) = (codes[r][k] >> t) & 1
 *   Kw = roundup(K, 128) / 32; padding bits are zero.
 * Bit decomposition is Eq. bitDecomposition; the 128-bit
 * run per plane matches the bmma k = 128 tile and the
 * "128c channels" remark (reading R3). */
size_t oracle_packed_words(int rows, int K, int bits)
{
    size_t Kw = ((size_t)K + 127) / 128 * 4;
    return (size_t)rows * bits * Kw;
}

int oracle_pack(const uint8_t *codes, int rows, int K, int bits, uint32_t *out)
{
    if (bits < 1 || bits > 8) return OR_ERR_BITS;
    if (rows < 0 || K < 0) return OR_ERR_SHAPE;
    if (!codes_in_range(codes, (size_t)rows * K, bits)) return OR_ERR_CODE;
    size_t Kw = ((size_t)K + 127) / 128 * 4;
    memset(out, 0, (size_t)rows * bits * Kw * sizeof(uint32_t));
    for (int r = 0; r < rows; r++)
        for (int t = 0; t < bits; t++)
            for (int k = 0; k < K; k++)
                if ((codes[(size_t)r * K + k] >> t) & 1)
                    out[((size_t)r * bits + t) * Kw + k / 32] |= (uint32_t)1 << (k % 32);
    return OR_OK;
}
