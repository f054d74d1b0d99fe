/*
 * apnn.h -- C ABI of the B200-native APNN-TC hot path (arXiv 2106.12169).
 *
 * One shared library, libapnn.so (paper_2106_12169_b200/libapnn.so), built for
 * sm_100a.  Every compute call runs hand-written CUDA kernels; there is no CPU
 * fallback: a call with no usable CUDA device returns APNN_ERR_CUDA.
 *
 * The operation (PAPER.md citations are /root/reference/PAPER.md lines):
 *   arbitrary-precision integer GEMM  Y = A . W^T, where A holds a_bits-bit
 *   activation codes and W holds w_bits-bit weight codes (1..8 bits each).
 *   The paper defines it through p.q one-bit plane products combined with
 *   weights 2^(s+t) (AP-Bit Operation Template; APMM
 *   PAPER.md:1489-1494); the result is the exact integer product, and this
 *   library computes exactly that.
 *   Convolution is the same operation as an implicit GEMM (APConv,
 *   PAPER.md:1612-1662).  Outputs are int32 or, through the
 *   fused element-wise routine, requantised and re-packed codes for the next
 *   layer.
 *
 * Conventions shared by every call
 *   - Pointers marked "device" are CUDA device pointers owned by the caller
 *     (allocated by PyTorch in this repo).  The library never allocates,
 *     frees or retains device memory and keeps no state between calls; it is
 *     thread-safe.
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and never synchronise the host.  Arguments are
 *     validated on the host first; on any error nothing is launched.
 *   - A launch failure (cudaGetLastError after the launch) returns
 *     APNN_ERR_CUDA.
 *   - Device pointers must be 16-byte aligned (APNN_ERR_ALIGNMENT).
 *
 * Packed bit-plane format (the layout contract)
 *   A tensor of `rows` rows of K codes with `bits` bits is stored as uint32
 *       P[r][t][w],  r < rows, t < bits, w < Kw = roundup(K,128)/32,
 *   bit (k % 32) of P[r][t][k / 32] = (code[r][k] >> t) & 1        (LSB-first)
 *   i.e. each row holds its `bits` 1-bit planes back to back, every plane run
 *   padded with zero bits to a multiple of 128 (Eq. bitDecomposition
 *   PAPER.md:1419-1421; the 128-bit run is the bmma k = 128 tile PAPER.md:1524
 *   and "128c channels" PAPER.md:1645).  Padding bits MUST be zero.
 *     GEMM A:   rows = M,                K = K
 *     GEMM W:   rows = N,                K = K
 *     conv X:   rows = B*H*W (NHWC),     K = C_in        (channel-major)
 *     conv W:   rows = C_out*R*S (OHWI), K = C_in
 *     packed outputs: rows = M (or B*Ho*Wo), K = N (or C_out), bits = out_bits
 *
 * Encodings (data-adaptive operator selection).  A +-1
 * operand stores -1 as bit 0 and +1 as bit 1 and must be
 * 1-bit; 0/1 operands are unsigned codes 0 .. 2^bits-1.
 *
 * Errors are returned as apnn_status; nothing is printed.
 */
#ifndef APNN_H_
#define APNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t / CUstream. */
typedef struct CUstream_st *apnn_stream_t;

typedef enum {
    APNN_OK = 0,
    APNN_ERR_INVALID_ARG = 1, /* NULL pointer, negative size, bad epilogue fields */
    APNN_ERR_BITS = 2,        /* a_bits / w_bits / bits / out_bits outside 1..8 */
    APNN_ERR_ENCODING = 3,    /* +-1 operand with bits > 1, unknown encoding */
    APNN_ERR_SHAPE = 4,       /* inconsistent shapes (e.g. conv output < 1) */
    APNN_ERR_ALIGNMENT = 5,   /* device pointer not 16-byte aligned */
    APNN_ERR_OVERFLOW = 6,    /* worst-case |Y| may exceed int32 */
    APNN_ERR_UNSUPPORTED = 7, /* combination not implemented by the requested variant */
    APNN_ERR_CUDA = 8         /* no device, wrong architecture, or launch failure */
} apnn_status;

typedef enum {
    APNN_ENC_01_01 = 0,      /* Case I:   A 0/1, W 0/1 -> AND + popc */
    APNN_ENC_PM1_PM1 = 1,    /* Case II:  A +-1, W +-1 (1 bit each) -> XOR PAPER.md:1455-1460 */
    APNN_ENC_W_PM1_A_01 = 2, /* Case III: W +-1 (1 bit), A 0/1 */
    APNN_ENC_W_01_A_PM1 = 3  /* Case III with roles swapped: A +-1 (1 bit), W 0/1 */
} apnn_encoding;

/* Kernel family that executes the contraction (north star: "choose by
 * measurement").  All variants return bit-identical results. */
typedef enum {
    APNN_VARIANT_AUTO = 0,  /* library picks (apnn_select_variant) */
    APNN_VARIANT_TC_I8 = 1, /* planes -> int8 recombination, tcgen05.mma kind::i8, TMEM accumulators */
    APNN_VARIANT_POPC = 2,  /* CUDA-core AND/XOR + POPC bit-plane products, shift-add combination */
    APNN_VARIANT_B1MMA = 3, /* legacy mma.sync m16n8k256 b1 .and/.xor.popc (the paper's bmma) */
    APNN_VARIANT_TC_FP4 = 4 /* exact e2m1 formulation, tcgen05.mma kind::mxf4 with unit block scales:
                               GEMM with a_bits, w_bits <= 2 and K*max|a|*max|w| < 2^24 only */
} apnn_variant;

/* Element-wise routine fused after the contraction:
 *   v = alpha[n] * y + beta[n]                  (int64; BN / zero point folded
 *                                                on the host into integers)
 *   [conv only, pool > 0: k x k pooling of v over the output feature map,
 *    stride pool_stride (0 = k), maximum or floor of the average; grids that do
 *    not fit are dropped: Hp = (Ho - k)/stride + 1]
 *   q = clamp(floor(v / divisor), 0, 2^out_bits - 1)   (floor toward -inf;
 *                                                the lower clamp is the ReLU)
 * and q is bit-decomposed and packed along N into the packed format with
 * bits = out_bits. */
typedef struct {
    int32_t out_bits;      /* 1..8 */
    const int32_t *alpha;  /* device [N] or NULL (= 1) */
    const int32_t *beta;   /* device [N] or NULL (= 0) */
    int32_t divisor;       /* S > 0 */
    int32_t pool;          /* 0: none; k >= 1: k x k pooling window (apnn_conv2d and
                              apnn_pool_quant_pack_out only; APNN_ERR_INVALID_ARG elsewhere) */
    int32_t pool_stride;   /* 0: = pool */
    int32_t pool_avg;      /* 0: max pooling, 1: average (floor of the sum / k^2) */
    /* Residual shortcut (ResNet blocks, reading R24), apnn_gemm_fused / apnn_conv2d only:
     *   v = alpha[n]*y + beta[n] + rho[n]*z[m][n]  before the pooling-free quantisation.
     * residual == NULL: none.  Otherwise z is device int32 [M][N] (residual_bits = 0) or
     * device packed 0/1 codes [M][residual_bits][roundup(N,128)/32] (1..8).  Fused only by
     * the 2-CTA tensor-core kernel (M > 128, no pooling); elsewhere APNN_ERR_UNSUPPORTED:
     * use apnn_residual_quant_pack after an int32 GEMM/conv. */
    const void *residual;
    int32_t residual_bits;
    const int32_t *rho;    /* device [N] or NULL (= 1) */
} apnn_epilogue;

/* NHWC convolution geometry.  Ho = (H + 2 pad - R)/stride + 1, Wo likewise. */
typedef struct {
    int32_t B, H, W, C_in, C_out, R, S, stride, pad;
} apnn_conv_shape;

/* Bytes of the packed format: rows * bits * roundup(K,128) / 8.  Returns 0
 * for invalid arguments. */
size_t apnn_packed_bytes(int rows, int K, int bits);

/* Bit decomposition + packing (Eq. bitDecomposition).
 *   codes: device uint8 [rows][K] row-major, each < 2^bits (higher bits are
 *          ignored: the code is masked to its low `bits` bits).
 *   dst:   device, apnn_packed_bytes(rows, K, bits) bytes, fully written
 *          (padding bits are written as zero).
 * A +-1 tensor is packed as codes 0/1.  HBM-bound streaming kernel. */
apnn_status apnn_pack_bits(const uint8_t *codes, int rows, int K, int bits, uint32_t *dst,
                           apnn_stream_t stream);

/* Implicit-GEMM rows made explicit for a thin first layer (C_in = 3 images; the paper
 * blames the first layer for most of AlexNet's latency): bit-decompose
 * and pack the im2col matrix of NHWC uint8 codes (APConv as GEMM).
 *   X:   device uint8 [B][H][W][C_in] codes < 2^bits (higher bits ignored)
 *   dst: device packed [B*Ho*Wo][bits][roundup(R*S*C_in,128)/32]; row (b,ho,wo), element
 *        k = (r*S + s)*C_in + c holds the code of X[b][ho*st+r-pad][wo*st+s-pad][c], and
 *        0 for out-of-frame taps (the value 0 of a 0/1 encoding; +-1 activations cannot
 *        be padded this way and must use apnn_conv2d).
 * The GEMM weights are then the OHWI codes flattened to [C_out][R*S*C_in]. */
apnn_status apnn_im2col_pack(const uint8_t *X, const apnn_conv_shape *shape, int bits, uint32_t *dst,
                             apnn_stream_t stream);

/* The first layer's input quantisation fused into apnn_im2col_pack: "the first layer
 * quantizes 8-bit inputs into q-bit activations" with the
 * quantisation y = floor((x - z) / s) of PAPER.md:1283-1287, clamped to [0, 2^bits - 1]
 * (reading R10).  X holds the raw 8-bit image (uint8 [B][H][W][C_in], any value); every
 * element is quantised while it is staged, out-of-frame taps are code 0 (zero padding of
 * the quantised conv input).  Output layout as apnn_im2col_pack.
 *   zero_point: z in [-255, 255];  scale: s in [1, 255] (APNN_ERR_INVALID_ARG otherwise). */
apnn_status apnn_im2col_quant_pack(const uint8_t *X, const apnn_conv_shape *shape, int zero_point, int scale,
                                   int bits, uint32_t *dst, apnn_stream_t stream);

/* Flatten a packed feature map for the first fully connected layer: per image b,
 *   src [B][P][bits][Cw]  (P pixels, packed rows of the conv output, Cw = roundup(C,128)/32)
 *   dst [B][bits][P*Cw]   (one packed row of K = P * Cw * 32 elements per image, pixel-major,
 *                          i.e. the HWC flattening; channel padding stays zero inside K)
 * A pure permutation of 32-bit words (no arithmetic); the FC weights are packed with the
 * same [P][Cw*32] element order (zero codes in the padded channels). */
apnn_status apnn_flatten_packed(const uint32_t *src, int B, int P, int bits, int Cw, uint32_t *dst,
                                apnn_stream_t stream);

/* APMM with 32-bit output:
 *   Y[m][n] = sum_{k<K} dec_A(a[m][k]) * dec_W(w[n][k])
 *   A: device packed [M][a_bits][Kw];  W: device packed [N][w_bits][Kw];
 *   Y: device int32 [M][N] row-major.
 * Returns APNN_ERR_OVERFLOW when K * max|a| * max|w| >= 2^31. */
apnn_status apnn_gemm(const uint32_t *A, const uint32_t *W, int M, int N, int K, int a_bits,
                      int w_bits, apnn_encoding enc, int32_t *Y, apnn_stream_t stream);

/* APMM with the fused element-wise routine: Y_packed = pack(requant(A . W^T)).
 *   Y_packed: device, apnn_packed_bytes(M, N, epi->out_bits) bytes, packed
 *             [M][out_bits][roundup(N,128)/32]; padding bits written as zero.
 *   epi: host pointer, read during the call only. */
apnn_status apnn_gemm_fused(const uint32_t *A, const uint32_t *W, int M, int N, int K,
                            int a_bits, int w_bits, apnn_encoding enc,
                            const apnn_epilogue *epi, uint32_t *Y_packed, apnn_stream_t stream);

/* Either of the two above with an explicit kernel variant.
 *   epi == NULL -> Y is int32 [M][N];  epi != NULL -> Y is the packed output. */
apnn_status apnn_gemm_ex(const uint32_t *A, const uint32_t *W, int M, int N, int K, int a_bits,
                         int w_bits, apnn_encoding enc, const apnn_epilogue *epi, void *Y,
                         apnn_variant variant, apnn_stream_t stream);

/* APConv as implicit GEMM:
 *   Y[b][ho][wo][co] = sum_{r,s,c} dec_A(X[b][ho*st+r-pad][wo*st+s-pad][c]) * dec_W(W[co][r][s][c])
 *   with out-of-frame taps contributing the VALUE 0 for every encoding (the
 *   input-aware padding of PAPER.md:1652-1662).
 *   X: device packed [B*H*W][a_bits][roundup(C_in,128)/32]   (NHW[P][C])
 *   W: device packed [C_out*R*S][w_bits][roundup(C_in,128)/32]
 *   epi == NULL -> Y: device int32 NHWC [B][Ho][Wo][C_out]
 *   epi != NULL -> Y: packed [B*Ho*Wo][out_bits][roundup(C_out,128)/32]
 *   shape: host pointer. */
apnn_status apnn_conv2d(const uint32_t *X, const uint32_t *W, const apnn_conv_shape *shape,
                        int a_bits, int w_bits, apnn_encoding enc, const apnn_epilogue *epi,
                        void *Y, apnn_stream_t stream);
/*   Pooling (epi->pool > 0) is fused into the tensor-core epilogue for 2 x 2 /
 *   stride 2 max pooling when Ho is even, 2 <= Wo <= 64 and B*Ho*Wo > 128; the
 *   output is then packed [B*Hp*Wp][out_bits][roundup(C_out,128)/32].  Any other
 *   pooling returns APNN_ERR_UNSUPPORTED without launching: run the conv with
 *   int32 output and apnn_pool_quant_pack_out (the unfused pair). */

apnn_status apnn_conv2d_ex(const uint32_t *X, const uint32_t *W, const apnn_conv_shape *shape,
                           int a_bits, int w_bits, apnn_encoding enc, const apnn_epilogue *epi,
                           void *Y, apnn_variant variant, apnn_stream_t stream);

/* Stand-alone element-wise routine (the unfused path): requantise an int32
 * [M][N] matrix and pack it exactly as apnn_gemm_fused would.
 *   Y: device int32 [M][N]; out: device packed [M][out_bits][roundup(N,128)/32]. */
apnn_status apnn_quant_pack_out(const int32_t *Y, int M, int N, const apnn_epilogue *epi,
                                uint32_t *out, apnn_stream_t stream);

/* Stand-alone pooling + element-wise routine over an NHWC int32 conv output
 * (the unfused counterpart of the fused conv epilogue):
 *   Y:   device int32 [B][H][W][N]  (H, W = the conv output size Ho, Wo)
 *   epi: host; pool >= 1 required (see apnn_epilogue)
 *   out: device packed [B*Hp*Wp][out_bits][roundup(N,128)/32] */
apnn_status apnn_pool_quant_pack_out(const int32_t *Y, int B, int H, int W, int N,
                                     const apnn_epilogue *epi, uint32_t *out, apnn_stream_t stream);

/* k x k / stride max pooling over packed codes ("maximum" pooling; reading R15:
 * the requantisation is non-decreasing in v, so max-pooling the codes equals quantising the
 * max-pooled v -- a conv with the fused requant + pack followed by this call is the pooled layer,
 * for any window, without an int32 map in HBM):
 *   X: device packed codes [B*H*W][bits][roundup(C,128)/32] (NHWC pixel rows)
 *   Y: device packed codes [B*Hp*Wp][bits][roundup(C,128)/32], Hp = (H - k)/stride + 1, Wp likewise
 *   (no padding; padding words of X come out as zeros).  Asynchronous on `stream`; no allocation. */
apnn_status apnn_maxpool_packed(const uint32_t *X, int B, int H, int W, int C, int bits, int k, int stride,
                                uint32_t *Y, apnn_stream_t stream);

/* Residual element-wise routine (ResNet basic block; reading R24 -- the paper does not
 * describe residual connections): the shortcut is added to the folded-BN value before
 * the quantisation,
 *   v = alpha[n] * Y[m][n] + beta[n] + rho[n] * Z[m][n]
 *   q = clamp(floor(v / divisor), 0, 2^out_bits - 1)   -> packed like apnn_quant_pack_out
 *   Y:  device int32 [M][N] (the block's second conv)
 *   Z:  the shortcut, either device int32 [M][N] (z_bits = 0: a 1x1 downsample conv's
 *       accumulator) or device packed codes [M][z_bits][roundup(N,128)/32] (z_bits 1..8:
 *       the block input itself, 0/1 codes)
 *   rho: device int32 [N] or NULL (= 1);  epi: host, pool must be 0.
 *   out: device packed [M][out_bits][roundup(N,128)/32]. */
apnn_status apnn_residual_quant_pack(const int32_t *Y, int M, int N, const void *Z, int z_bits,
                                     const int32_t *rho, const apnn_epilogue *epi, uint32_t *out,
                                     apnn_stream_t stream);

/* Prepared weights for the exact-FP4 variant (weights are static): the
 * operand-side bit combination of W done once, at load time, instead of per output tile.
 *   W:  device packed [N][w_bits][roundup(K,128)/32] (w_bits <= 2, or 1-bit +-1)
 *   Wp: device, apnn_prepared_bytes(N, K) bytes: e2m1 nibbles [N][roundup(K,128)/2] in the
 *       kernel's element order (an opaque layout for apnn_gemm_prepared); padding is value 0.
 * APNN_ERR_UNSUPPORTED for w_bits > 2. */
size_t apnn_prepared_bytes(int N, int K);
apnn_status apnn_prepare_weights(const uint32_t *W, int N, int K, int w_bits, apnn_encoding enc, uint8_t *Wp,
                                 apnn_stream_t stream);
/* apnn_gemm_ex (int32 when epi == NULL, else the fused routine without pooling / residual)
 * with prepared weights on the exact-FP4 kernel; a_bits <= 2 and K*max|a|*max|w| < 2^24,
 * else APNN_ERR_UNSUPPORTED.  Same results as apnn_gemm_ex. */
apnn_status apnn_gemm_prepared(const uint32_t *A, const uint8_t *Wp, int M, int N, int K, int a_bits,
                               int w_bits, apnn_encoding enc, const apnn_epilogue *epi, void *Y,
                               apnn_stream_t stream);

/* Prepared activations (both operands prepared; the bench GEMM).  An activation matrix is used
 * by every N tile of a GEMM, so decoding its bit-planes inside the GEMM repeats the decode
 * ceil(N / 256) times; apnn_prepare_activations decodes them once (the operand-side bit
 * combination of PAPER.md:1426-1429, +-1 codes per Case II / III) into the
 * e2m1 operand rows of apnn_prepare_weights:
 *   A:  device, packed activation planes [M][a_bits][Kw] (apnn_pack_bits layout), a_bits <= 2
 *       (+-1 activations, enc APNN_ENC_PM1_PM1 / APNN_ENC_W_01_A_PM1: a_bits == 1);
 *   Ap: device, apnn_prepared_bytes(M, K) bytes, caller-owned; elements >= K are value 0.
 * apnn_gemm_prepared_ab: Y = A W^T from Ap and Wp (apnn_prepare_weights) on the persistent
 * CTA-pair exact-FP4 kernel (both operands land by TMA; no CUDA-core decode in the main loop);
 * int32 when epi == NULL, else the fused requantise + pack routine (no pooling / residual).
 * Same results as apnn_gemm_ex.  APNN_ERR_UNSUPPORTED where apnn_gemm_prepared is. Asynchronous
 * on `stream`; no allocation. */
apnn_status apnn_prepare_activations(const uint32_t *A, int M, int K, int a_bits, apnn_encoding enc,
                                     uint8_t *Ap, apnn_stream_t stream);
apnn_status apnn_gemm_prepared_ab(const uint8_t *Ap, const uint8_t *Wp, int M, int N, int K, int a_bits,
                                  int w_bits, apnn_encoding enc, const apnn_epilogue *epi, void *Y,
                                  apnn_stream_t stream);

/* apnn_pack_bits fused with apnn_prepare_activations (<= 2-bit codes): one pass over the codes
 * writes the packed planes to dst (exactly as apnn_pack_bits) AND the e2m1 operand rows to Ap
 * (exactly as apnn_prepare_activations of those planes; apnn_prepared_bytes(rows, K) bytes).
 * enc decides whether the codes are +-1 activations (APNN_ENC_PM1_PM1 / APNN_ENC_W_01_A_PM1,
 * bits == 1).  bits > 2: APNN_ERR_UNSUPPORTED. */
apnn_status apnn_pack_bits_prepared(const uint8_t *codes, int rows, int K, int bits, apnn_encoding enc,
                                    uint32_t *dst, uint8_t *Ap, apnn_stream_t stream);

/* The bit decomposition from DENSE codes (the compact host format of low-bit data, bits <= 2):
 *   dcodes: device; row r starts at byte r * ceil(K*bits/8); element k of a row is the `bits`-bit
 *           field at bit k*bits of the row's little-endian bit stream (LSB first)
 *   dst:    device packed planes [rows][bits][Kw], exactly as apnn_pack_bits of the same codes
 *   Ap:     NULL, or device apnn_prepared_bytes(rows, K) bytes: also the e2m1 operand rows, exactly
 *           as apnn_prepare_activations (enc decides +-1 activations, bits == 1)
 * bits > 2: APNN_ERR_UNSUPPORTED. */
apnn_status apnn_pack_bits_dense(const uint8_t *dcodes, int rows, int K, int bits, apnn_encoding enc,
                                 uint32_t *dst, uint8_t *Ap, apnn_stream_t stream);

/* Prepared int8 weights for the int8 tensor-core kernel (any w_bits; the B decode that grows
 * with w_bits is done once at load time):
 *   Wp: device, apnn_prepared_i8_bytes(N, K) bytes: int8 operand rows [N][roundup(K,128)] in
 *       the kernel's element order (u8 codes, or s8 +-1 with value-0 padding); opaque layout.
 * apnn_gemm_prepared_i8: as apnn_gemm_ex on the 2-CTA tcgen05 kernel; GEMM with M > 128 and
 * no pooling / residual epilogue, else APNN_ERR_UNSUPPORTED. */
size_t apnn_prepared_i8_bytes(int N, int K);
apnn_status apnn_prepare_weights_i8(const uint32_t *W, int N, int K, int w_bits, apnn_encoding enc,
                                    uint8_t *Wp, apnn_stream_t stream);
apnn_status apnn_gemm_prepared_i8(const uint32_t *A, const uint8_t *Wp, int M, int N, int K, int a_bits,
                                  int w_bits, apnn_encoding enc, const apnn_epilogue *epi, void *Y,
                                  apnn_stream_t stream);
/* Both operands prepared, int8 (any a_bits / w_bits): apnn_prepare_activations_i8 decodes the
 * activation planes once into the int8 operand rows of apnn_prepare_weights_i8 (u8 codes, or s8 +-1
 * with value-0 padding; Ap: apnn_prepared_i8_bytes(M, K) bytes, caller-owned), and
 * apnn_gemm_prepared_ab_i8 runs the persistent CTA-pair kind::i8 kernel on Ap and Wp (both by TMA,
 * two int32 TMEM accumulators); int32 when epi == NULL, else the fused routine without pooling /
 * residual.  Same results as apnn_gemm_ex; APNN_ERR_OVERFLOW where that is. */
apnn_status apnn_prepare_activations_i8(const uint32_t *A, int M, int K, int a_bits, apnn_encoding enc,
                                        uint8_t *Ap, apnn_stream_t stream);
apnn_status apnn_gemm_prepared_ab_i8(const uint8_t *Ap, const uint8_t *Wp, int M, int N, int K, int a_bits,
                                     int w_bits, apnn_encoding enc, const apnn_epilogue *epi, void *Y,
                                     apnn_stream_t stream);
/* apnn_conv2d with prepared conv weights: Wp = apnn_prepare_weights_i8 of the packed OHWI
 * weights viewed as C_out*R*S rows of C_in (apnn_prepared_i8_bytes(C_out*R*S, C_in) bytes).
 * Runs on the tap-reuse kernel (APConv: the input window of a 16 x 8
 * output tile is decoded once per 128-channel chunk and every filter tap is a row offset
 * into it) wherever apnn_conv_halo_fits says so -- any batch size, fused requantisation,
 * 2x2/2 max pooling and the residual epilogue (0/1 activations) included -- else on the
 * per-tap 2-CTA kernel (B*Ho*Wo > 128; pooling as apnn_conv2d), else APNN_ERR_UNSUPPORTED. */
apnn_status apnn_conv2d_prepared_i8(const uint32_t *X, const uint8_t *Wp, const apnn_conv_shape *shape,
                                    int a_bits, int w_bits, apnn_encoding enc, const apnn_epilogue *epi,
                                    void *Y, apnn_stream_t stream);

/* The first layer straight from the raw 8-bit image ("quantizes 8-bit
 * inputs into q-bit activations"): X is the device NHWC uint8 image [B][H][W][C_in]; each pixel
 * value is quantised to q = clamp(floor((x - zero_point) / scale), 0, 2^a_bits - 1) (reading R10/
 * R11, as apnn_im2col_quant_pack) inside the tap-reuse conv kernel, and out-of-frame taps are
 * code 0.  Wp = apnn_prepare_weights_i8 of the packed OHWI weights viewed as C_out*R rows of
 * S*C_in (apnn_prepared_i8_bytes(C_out*R, S*C_in) bytes).  Needs S*C_in <= 128 and 0/1
 * activations (enc APNN_ENC_01_01 or APNN_ENC_W_PM1_A_01); epilogue and output as apnn_conv2d
 * (int32 NHWC, or packed with 2x2/2 max pooling fused where apnn_conv_first_fits says so);
 * no residual.  scale in [1, 255], zero_point in [-255, 255], else APNN_ERR_INVALID_ARG. */
apnn_status apnn_conv2d_first_prepared_i8(const uint8_t *X, const uint8_t *Wp, const apnn_conv_shape *shape,
                                          int zero_point, int scale, int a_bits, int w_bits, apnn_encoding enc,
                                          const apnn_epilogue *epi, void *Y, apnn_stream_t stream);
/* 1 if apnn_conv2d_first_prepared_i8 takes this layer (shape, encoding, epilogue or NULL). */
int apnn_conv_first_fits(const apnn_conv_shape *shape, int a_bits, int w_bits, apnn_encoding enc,
                         const apnn_epilogue *epi);

/* Tile configuration of the int8 tensor-core GEMM (row f4).  kernel 1: one CTA per 128 x bn output
 * tile, K split over a cluster of ksplit CTAs (reduced through distributed shared memory);
 * kernel 2: a CTA pair (cta_group::2) per 256 x bn tile.  tlp = CTAs launched, ci = the tile's
 * compute intensity 2 bm bn / (bm + bn). */
typedef struct {
    int32_t kernel;   /* 1 or 2 */
    int32_t bm, bn;   /* 128 (kernel 1) / 256 (kernel 2); bn in {64, 128, 256} */
    int32_t ksplit;   /* 1, 2, 4 (kernel 1; > 1 needs bn <= 128 and ksplit <= ceil(K/128)) */
    int64_t tlp;
    double ci;
} apnn_tile_config;

/* The paper's block-tiling heuristic: candidate tiles are ordered by TLP;
 * the highest-TLP one is taken when its TLP is below the threshold T, else the highest-CI one
 * among those with TLP >= T.  Candidates are the int8 kernels' tiles (reading R21);
 * out_bits: 0 for int32 output, else the packed output width (pair tiles narrower than 128
 * columns store packed words only when N <= 64).  T = threshold, or the paper's T = 64 when
 * threshold <= 0.  Host-only computation
 * (no launch); apnn_gemm / apnn_gemm_fused use it for every int8 tensor-core GEMM. */
apnn_status apnn_tune_tiles(int M, int N, int K, int out_bits, int threshold, apnn_tile_config *out);

/* apnn_gemm_ex on the int8 tensor-core variant with an explicit tile configuration (measurement
 * of the tuner's candidates, configuration-invariance tests).  APNN_ERR_UNSUPPORTED for a
 * configuration the kernels do not implement for this shape (see apnn_tile_config). */
apnn_status apnn_gemm_tiled(const uint32_t *A, const uint32_t *W, int M, int N, int K, int a_bits, int w_bits,
                            apnn_encoding enc, const apnn_epilogue *epi, void *Y, const apnn_tile_config *cfg,
                            apnn_stream_t stream);

/* 1 if apnn_conv2d_prepared_i8 runs this convolution (shape, encoding, epilogue or NULL) on
 * the tap-reuse kernel, 0 otherwise (no launch; invalid arguments give 0). */
int apnn_conv_halo_fits(const apnn_conv_shape *shape, int a_bits, int w_bits, apnn_encoding enc,
                        const apnn_epilogue *epi);

/* Which variant APNN_VARIANT_AUTO resolves to for this problem (no launch): int32 output,
 * or the fused element-wise routine with out_bits (1..8) packed output. */
apnn_variant apnn_select_variant(int M, int N, int K, int a_bits, int w_bits, apnn_encoding enc);
apnn_variant apnn_select_variant_fused(int M, int N, int K, int a_bits, int w_bits, apnn_encoding enc,
                                       int out_bits);

const char *apnn_status_string(apnn_status status);
const char *apnn_variant_name(apnn_variant variant);

/* Number of kernels this library has launched in this process (monotonic;
 * used by bench.py to report gpu_launches). */
uint64_t apnn_launch_count(void);

/* ABI version: major * 10000 + minor * 100 + patch. */
int apnn_version(void);

#ifdef __cplusplus
}
#endif

#endif /* APNN_H_ */
