// apnn.cu -- the C ABI (include/apnn.h): host-side validation and dispatch.
//
// Nothing here computes results: every call validates its arguments, builds
// the kernel parameters and launches one of the sm_100a kernels on the caller's
// stream.  There is no CPU path; a missing/unsupported device is an error.
#include <atomic>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace apnn {

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

cudaError_t launch_pack_bits(const uint8_t* codes, int rows, int K, int bits, uint32_t* dst, int sms,
                             cudaStream_t s, uint8_t* prep = nullptr, bool pm1 = false);
cudaError_t launch_pack_dense(const uint8_t* codes, int rows, int K, int bits, uint32_t* dst, int sms,
                              cudaStream_t s, uint8_t* prep, bool pm1);
cudaError_t launch_quant_pack(const int32_t* Y, int M, int N, const Epi& e, uint32_t* out, int sms,
                              cudaStream_t s);
cudaError_t launch_maxpool_packed(const uint32_t* X, int B, int H, int W, int C, int bits, int k, int stride,
                                  uint32_t* Y, int sms, cudaStream_t s);
cudaError_t launch_pool_quant_pack(const int32_t* Y, int B, int H, int W, int N, const Epi& e, uint32_t* out,
                                  int sms, cudaStream_t s);
bool tc_i8_pool_fusable(const Geom& g, const Epi& e);
cudaError_t launch_residual_quant_pack(const int32_t* Y, int M, int N, const void* Z, int z_bits,
                                       const int32_t* rho, const Epi& e, uint32_t* out, int sms, cudaStream_t s);
cudaError_t launch_flatten_packed(const uint32_t* src, int B, int P, int bits, int Cw, uint32_t* dst, int sms,
                                  cudaStream_t s);
cudaError_t launch_im2col_pack(const uint8_t* X, int B, int H, int W, int C, int R, int S, int stride, int pad,
                               int Ho, int Wo, int bits, uint32_t* dst, int sms, cudaStream_t s, int qz = 0,
                               int qs = 0);
cudaError_t launch_popc(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                        cudaStream_t s);
cudaError_t launch_b1mma(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                         cudaStream_t s);
cudaError_t launch_tc_i8(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                         int sms, cudaStream_t s);
bool tc_i8_supports(const Geom& g);
bool tc_fp4_supports(const Geom& g);
cudaError_t launch_tc_fp4(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                          cudaStream_t s);
cudaError_t launch_tc_fp4_prepared(const uint32_t* A, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                   cudaStream_t s);
cudaError_t launch_prepare_weights(const uint32_t* W, int N, int K, int w_bits, int enc, uint8_t* out, int sms,
                                   cudaStream_t s);
cudaError_t launch_tc_fp4_pair_prepared_ab(const uint8_t* Ap, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                           int sms, cudaStream_t s);
cudaError_t launch_tc_i8_prepared_ab(const uint8_t* Ap, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                     int sms, cudaStream_t s);
cudaError_t launch_tc_fp4_pair_prepared(const uint32_t* A, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                        int sms, cudaStream_t s);
cudaError_t launch_prepare_weights_i8(const uint32_t* W, int N, int K, int w_bits, int enc, uint8_t* out, int sms,
                                      cudaStream_t s);
cudaError_t launch_tc_i8_prepared(const uint32_t* A, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y,
                                  int sms, cudaStream_t s);
bool b1mma_supports(const Geom& g);
bool conv_halo_supports(const Geom& g, const Epi& e);
cudaError_t launch_conv_halo(const uint32_t* X, const uint8_t* Wp, const Geom& g, const Epi& e, void* Y, int sms,
                             cudaStream_t s);

cudaError_t launch_tc_i8_tiled(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                               const TileCfg& cfg, int sms, cudaStream_t s);
bool conv_first_supports(const Geom& g, const Epi& e, int S_raw, int C_raw);
cudaError_t launch_conv_first(const uint8_t* X, const uint8_t* Wp, const Geom& g, const Epi& e, int qz, int qs,
                              int S_raw, int C_raw, void* Y, int sms, cudaStream_t s);

// APNN_CONV_HALO=0 (read once) keeps prepared-weight convolutions on the per-tap 2-CTA
// kernel (A/B measurements); default: the tap-reuse kernel wherever it fits
static bool conv_halo_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_CONV_HALO");
        v = s ? atoi(s) : 1;
    }
    return v != 0;
}

// ---- device properties (cached per device ordinal)
struct DevInfo {
    bool ok;
    int sms;
};
static std::mutex g_dev_mu;
static DevInfo g_dev[64];
static bool g_dev_init[64];

static apnn_status device_info(DevInfo* out) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return APNN_ERR_CUDA;
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_dev_init[dev]) {
        cudaDeviceProp p;
        DevInfo d{false, 0};
        if (cudaGetDeviceProperties(&p, dev) == cudaSuccess) {
            d.ok = (p.major == 10 && p.minor == 0);  // sm_100 (B200); the cubin is sm_100a only
            d.sms = p.multiProcessorCount;
        } else {
            cudaGetLastError();
        }
        g_dev[dev] = d;
        g_dev_init[dev] = true;
    }
    *out = g_dev[dev];
    return out->ok ? APNN_OK : APNN_ERR_CUDA;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static apnn_status check_bits_enc(int a_bits, int w_bits, int enc) {
    if (a_bits < 1 || a_bits > 8 || w_bits < 1 || w_bits > 8) return APNN_ERR_BITS;
    switch (enc) {
    case APNN_ENC_01_01: return APNN_OK;
    case APNN_ENC_PM1_PM1: return (a_bits == 1 && w_bits == 1) ? APNN_OK : APNN_ERR_ENCODING;
    case APNN_ENC_W_PM1_A_01: return (w_bits == 1) ? APNN_OK : APNN_ERR_ENCODING;
    case APNN_ENC_W_01_A_PM1: return (a_bits == 1) ? APNN_OK : APNN_ERR_ENCODING;
    default: return APNN_ERR_ENCODING;
    }
}

// worst case |y| = K * max|a| * max|w| must stay below 2^31
static apnn_status check_overflow(long long K, int a_bits, int w_bits, int enc) {
    long long ma = (enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1) ? 1 : ((1LL << a_bits) - 1);
    long long mw = (enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_PM1_A_01) ? 1 : ((1LL << w_bits) - 1);
    return (K * ma * mw > 2147483647LL) ? APNN_ERR_OVERFLOW : APNN_OK;
}

static apnn_status make_epi(const apnn_epilogue* epi, Epi* e) {
    std::memset(e, 0, sizeof(*e));
    if (!epi) return APNN_OK;
    if (epi->out_bits < 1 || epi->out_bits > 8) return APNN_ERR_BITS;
    if (epi->divisor <= 0 || epi->pool < 0 || epi->pool_stride < 0 || (epi->pool_avg != 0 && epi->pool_avg != 1))
        return APNN_ERR_INVALID_ARG;
    if ((epi->alpha && !aligned16(epi->alpha)) || (epi->beta && !aligned16(epi->beta)))
        return APNN_ERR_ALIGNMENT;
    e->alpha = epi->alpha;
    e->beta = epi->beta;
    e->S = epi->divisor;
    e->out_bits = epi->out_bits;
    e->qmax = (1 << epi->out_bits) - 1;
    e->invS = 1.0f / (float)epi->divisor;
    e->pool = epi->pool;
    e->pool_stride = epi->pool ? (epi->pool_stride ? epi->pool_stride : epi->pool) : 0;
    e->pool_avg = epi->pool_avg;
    if (epi->residual) {
        if (epi->residual_bits < 0 || epi->residual_bits > 8) return APNN_ERR_BITS;
        if (!aligned16(epi->residual) || (epi->rho && !aligned16(epi->rho))) return APNN_ERR_ALIGNMENT;
        if (epi->pool) return APNN_ERR_INVALID_ARG;
    }
    e->res = epi->residual;
    e->res_bits = epi->residual_bits;
    e->rho = epi->rho;
    return APNN_OK;
}

// AUTO dispatch (measured, scripts/fp4_time.py, profiles/r01_fp4.json): the exact FP4
// formulation wins every GEMM with operands <= 2 bits and at least 64 tiles of 128 x 256
// (fused output, or int32 output with N >= 256); the int8 tensor-core variant everything else
// (conv, wider codes, narrow int32 outputs, small-M split-K, residual / pooling epilogues).
static bool fp4_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_FP4");
        v = s ? atoi(s) : 1;
    }
    return v != 0;
}

static int fp4_kernel_choice() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_FP4_KERNEL");
        v = s ? atoi(s) : 0;
    }
    return v;
}

static apnn_variant resolve(apnn_variant v, const Geom& g, const Epi* e = nullptr) {
    if (v != APNN_VARIANT_AUTO) return v;
    const bool fused = e && e->out_bits > 0;
    // the FP4 kernel is one CTA per 128 x 256 tile without split-K: require enough tiles to
    // fill the SMs, else the int8 variant's split-K clusters win (VGG FC at batch 256)
    const long long fp4_tiles = (long long)((g.M + 127) / 128) * ((g.N + 255) / 256);
    // int32 outputs: only wide ones (the models' first-layer GEMMs, N = 64..96, measured faster
    // on the int8 pair kernel)
    if (fp4_enabled() && tc_fp4_supports(g) && fp4_tiles >= 64 && !(e && (e->res || e->pool)) &&
        (fused || g.N >= 256))
        return APNN_VARIANT_TC_FP4;
    // latency-scale GEMMs with 1-bit weights and <= 2-bit activations (the paper's FC layers):
    // the warp-level popc/shuffle kernel beats every tensor-core launch up to ~2^28 plane-bit
    // MACs (profiles/r02_popc_time.json: M = 64, N = K = 1024 w1a2 4.1 us vs 8.1 us, w1a1 3.4 vs
    // 7.8; 128^3 w1a2 3.2 vs 5.1; M = 1, N = K = 4096 w1a2 5.8 vs 15.2); wider weights loop over
    // their planes and lose
    if (!g.conv && g.w_bits == 1 && g.a_bits <= 2 && g.M <= 256 &&
        (long long)g.M * g.N * g.K * g.a_bits <= (1LL << 28) && !(e && (e->res || e->pool)))
        return APNN_VARIANT_POPC;
    if (tc_i8_supports(g)) return APNN_VARIANT_TC_I8;
    return APNN_VARIANT_POPC;
}

static apnn_status run(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                       apnn_variant variant, cudaStream_t s) {
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    if (g.M == 0 || g.N == 0) return APNN_OK;
    cudaError_t err;
    switch (resolve(variant, g, &e)) {
    case APNN_VARIANT_TC_I8:
        if (!tc_i8_supports(g)) return APNN_ERR_UNSUPPORTED;
        err = launch_tc_i8(A, W, g, e, Y, d.sms, s);
        break;
    case APNN_VARIANT_POPC: err = launch_popc(A, W, g, e, Y, s); break;
    case APNN_VARIANT_TC_FP4:
        if (!tc_fp4_supports(g) || e.res || e.pool) return APNN_ERR_UNSUPPORTED;
        err = launch_tc_fp4(A, W, g, e, Y, s);
        break;
    case APNN_VARIANT_B1MMA:
        if (!b1mma_supports(g)) return APNN_ERR_UNSUPPORTED;
        err = launch_b1mma(A, W, g, e, Y, s);
        break;
    default: return APNN_ERR_INVALID_ARG;
    }
    if (err == cudaErrorNotSupported) return APNN_ERR_UNSUPPORTED;  // e.g. residual epilogue off the 2-CTA kernel
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

static void gemm_geom(Geom* g, int M, int N, int K, int a_bits, int w_bits, int enc) {
    std::memset(g, 0, sizeof(*g));
    g->M = M; g->N = N; g->K = K;
    g->a_bits = a_bits; g->w_bits = w_bits; g->enc = enc;
    g->Cw = (K + 127) / 128 * 4;
    g->CB = g->Cw / 4;
    g->C = K;
    g->RS = 1;
    g->nchunks = g->CB;
    g->S = 1; g->stride = 1;
}

}  // namespace apnn

using namespace apnn;

extern "C" {

size_t apnn_packed_bytes(int rows, int K, int bits) {
    if (rows < 0 || K < 0 || bits < 1 || bits > 8) return 0;
    return (size_t)rows * (size_t)bits * (((size_t)K + 127) / 128 * 16);
}

apnn_status apnn_pack_bits(const uint8_t* codes, int rows, int K, int bits, uint32_t* dst,
                           apnn_stream_t stream) {
    if (rows < 0 || K < 0) return APNN_ERR_SHAPE;
    if (bits < 1 || bits > 8) return APNN_ERR_BITS;
    if ((rows > 0 && K > 0 && !codes) || (rows > 0 && !dst)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(dst)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    cudaError_t err = launch_pack_bits(codes, rows, K, bits, dst, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_pack_bits_prepared(const uint8_t* codes, int rows, int K, int bits, apnn_encoding enc,
                                    uint32_t* dst, uint8_t* Ap, apnn_stream_t stream) {
    if (rows < 0 || K < 0) return APNN_ERR_SHAPE;
    if (bits < 1 || bits > 8) return APNN_ERR_BITS;
    if (enc < 0 || enc > 3) return APNN_ERR_ENCODING;
    const bool apm = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1;
    if (apm && bits != 1) return APNN_ERR_ENCODING;
    if (bits > 2) return APNN_ERR_UNSUPPORTED;
    if ((rows > 0 && K > 0 && !codes) || (rows > 0 && (!dst || !Ap))) return APNN_ERR_INVALID_ARG;
    if (!aligned16(dst) || !aligned16(Ap)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    cudaError_t err = launch_pack_bits(codes, rows, K, bits, dst, d.sms, (cudaStream_t)stream, Ap, apm);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_pack_bits_dense(const uint8_t* dcodes, int rows, int K, int bits, apnn_encoding enc,
                                 uint32_t* dst, uint8_t* Ap, apnn_stream_t stream) {
    if (rows < 0 || K < 0) return APNN_ERR_SHAPE;
    if (bits < 1 || bits > 8) return APNN_ERR_BITS;
    if (enc < 0 || enc > 3) return APNN_ERR_ENCODING;
    const bool apm = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1;
    if (apm && bits != 1) return APNN_ERR_ENCODING;
    if (bits > 2) return APNN_ERR_UNSUPPORTED;
    if ((long long)K * bits > 2147483647LL) return APNN_ERR_SHAPE;
    if ((rows > 0 && K > 0 && !dcodes) || (rows > 0 && !dst)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(dst) || !aligned16(Ap)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    cudaError_t err = launch_pack_dense(dcodes, rows, K, bits, dst, d.sms, (cudaStream_t)stream, Ap, apm);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_flatten_packed(const uint32_t* src, int B, int P, int bits, int Cw, uint32_t* dst,
                                apnn_stream_t stream) {
    if (B < 0 || P < 1 || Cw < 1 || (Cw & 3)) return APNN_ERR_SHAPE;
    if (bits < 1 || bits > 8) return APNN_ERR_BITS;
    if ((long long)P * Cw * 32 > 2147483647LL) return APNN_ERR_SHAPE;
    if (B > 0 && (!src || !dst)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(src) || !aligned16(dst)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    cudaError_t err = launch_flatten_packed(src, B, P, bits, Cw, dst, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

static apnn_status im2col_impl(const uint8_t* X, const apnn_conv_shape* shp, int bits, uint32_t* dst, int qz,
                               int qs, apnn_stream_t stream);

apnn_status apnn_im2col_pack(const uint8_t* X, const apnn_conv_shape* shp, int bits, uint32_t* dst,
                             apnn_stream_t stream) {
    return im2col_impl(X, shp, bits, dst, 0, 0, stream);
}

apnn_status apnn_im2col_quant_pack(const uint8_t* X, const apnn_conv_shape* shp, int zero_point, int scale,
                                   int bits, uint32_t* dst, apnn_stream_t stream) {
    if (scale < 1 || scale > 255 || zero_point < -255 || zero_point > 255) return APNN_ERR_INVALID_ARG;
    return im2col_impl(X, shp, bits, dst, zero_point, scale, stream);
}

static apnn_status im2col_impl(const uint8_t* X, const apnn_conv_shape* shp, int bits, uint32_t* dst, int qz,
                               int qs, apnn_stream_t stream) {
    if (!shp) return APNN_ERR_INVALID_ARG;
    const apnn_conv_shape c = *shp;
    if (c.B < 0 || c.H < 1 || c.W < 1 || c.C_in < 1 || c.R < 1 || c.S < 1 || c.stride < 1 || c.pad < 0)
        return APNN_ERR_SHAPE;
    if (bits < 1 || bits > 8) return APNN_ERR_BITS;
    if (c.H + 2 * c.pad < c.R || c.W + 2 * c.pad < c.S) return APNN_ERR_SHAPE;
    const int Ho = (c.H + 2 * c.pad - c.R) / c.stride + 1;
    const int Wo = (c.W + 2 * c.pad - c.S) / c.stride + 1;
    const long long rows = (long long)c.B * Ho * Wo, K = (long long)c.R * c.S * c.C_in;
    if (rows > 2147483647LL || K > 2147483647LL - 127) return APNN_ERR_SHAPE;
    if (rows > 0 && (!X || !dst)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(dst)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    cudaError_t err = launch_im2col_pack(X, c.B, c.H, c.W, c.C_in, c.R, c.S, c.stride, c.pad, Ho, Wo, bits, dst,
                                         d.sms, (cudaStream_t)stream, qz, qs);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_gemm_ex(const uint32_t* A, const uint32_t* W, int M, int N, int K, int a_bits,
                         int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                         apnn_variant variant, apnn_stream_t stream) {
    if (M < 0 || N < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if ((M > 0 && K > 0 && !A) || (N > 0 && K > 0 && !W) || (M > 0 && N > 0 && !Y))
        return APNN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(W) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    if ((st = check_overflow(K, a_bits, w_bits, enc)) != APNN_OK) return st;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if (e.pool) return APNN_ERR_INVALID_ARG;  // pooling is a conv epilogue
    if ((unsigned)variant > (unsigned)APNN_VARIANT_TC_FP4) return APNN_ERR_INVALID_ARG;
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    if (e.res && (resolve(variant, g, &e) != APNN_VARIANT_TC_I8 || M <= 128 || enc == APNN_ENC_PM1_PM1 ||
                  enc == APNN_ENC_W_01_A_PM1))
        return APNN_ERR_UNSUPPORTED;  // fused residual: 2-CTA int8 kernel, 0/1 activations
    return run(A, W, g, e, Y, variant, (cudaStream_t)stream);
}

size_t apnn_prepared_bytes(int N, int K) {
    if (N < 0 || K < 0) return 0;
    return (size_t)N * (((size_t)K + 127) / 128 * 64);
}

apnn_status apnn_prepare_weights(const uint32_t* W, int N, int K, int w_bits, apnn_encoding enc, uint8_t* Wp,
                                 apnn_stream_t stream) {
    if (N < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = APNN_OK;
    if (w_bits < 1 || w_bits > 8) return APNN_ERR_BITS;
    if (enc < 0 || enc > 3) return APNN_ERR_ENCODING;
    const bool wpm = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_PM1_A_01;
    if (wpm && w_bits != 1) return APNN_ERR_ENCODING;
    if (w_bits > 2) return APNN_ERR_UNSUPPORTED;
    if (N > 0 && K > 0 && (!W || !Wp)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(W) || !aligned16(Wp)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    cudaError_t err = launch_prepare_weights(W, N, K, w_bits, enc, Wp, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_gemm_prepared(const uint32_t* A, const uint8_t* Wp, int M, int N, int K, int a_bits, int w_bits,
                               apnn_encoding enc, const apnn_epilogue* epi, void* Y, apnn_stream_t stream) {
    if (M < 0 || N < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if ((M > 0 && K > 0 && !A) || (N > 0 && K > 0 && !Wp) || (M > 0 && N > 0 && !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(Wp) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if (e.pool || e.res) return APNN_ERR_INVALID_ARG;
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    if (!tc_fp4_supports(g)) return APNN_ERR_UNSUPPORTED;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (M == 0 || N == 0) return APNN_OK;
    // M > 128: the persistent CTA-pair kernel (gemm_fp4_pair.cu); else the one-CTA kernel.
    // APNN_FP4_KERNEL=1 (read once) forces the one-CTA kernel for A/B measurements.
    cudaError_t err = (M > 128 && fp4_kernel_choice() != 1)
                          ? launch_tc_fp4_pair_prepared(A, Wp, g, e, Y, d.sms, (cudaStream_t)stream)
                          : launch_tc_fp4_prepared(A, Wp, g, e, Y, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_prepare_activations(const uint32_t* A, int M, int K, int a_bits, apnn_encoding enc, uint8_t* Ap,
                                     apnn_stream_t stream) {
    if (M < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = APNN_OK;
    if (a_bits < 1 || a_bits > 8) return APNN_ERR_BITS;
    if (enc < 0 || enc > 3) return APNN_ERR_ENCODING;
    const bool apm = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1;
    if (apm && a_bits != 1) return APNN_ERR_ENCODING;
    if (a_bits > 2) return APNN_ERR_UNSUPPORTED;
    if (M > 0 && K > 0 && (!A || !Ap)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(Ap)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    // the operand rows of apnn_prepare_weights, with the +-1 decision taken on A's side
    cudaError_t err = launch_prepare_weights(A, M, K, a_bits, apm ? APNN_ENC_PM1_PM1 : APNN_ENC_01_01, Ap, d.sms,
                                             (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_gemm_prepared_ab(const uint8_t* Ap, const uint8_t* Wp, int M, int N, int K, int a_bits, int w_bits,
                                  apnn_encoding enc, const apnn_epilogue* epi, void* Y, apnn_stream_t stream) {
    if (M < 0 || N < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if ((M > 0 && K > 0 && !Ap) || (N > 0 && K > 0 && !Wp) || (M > 0 && N > 0 && !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(Ap) || !aligned16(Wp) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if (e.pool || e.res) return APNN_ERR_INVALID_ARG;
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    if (!tc_fp4_supports(g)) return APNN_ERR_UNSUPPORTED;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (M == 0 || N == 0) return APNN_OK;
    cudaError_t err = launch_tc_fp4_pair_prepared_ab(Ap, Wp, g, e, Y, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_prepare_activations_i8(const uint32_t* A, int M, int K, int a_bits, apnn_encoding enc, uint8_t* Ap,
                                        apnn_stream_t stream) {
    if (M < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = APNN_OK;
    if (a_bits < 1 || a_bits > 8) return APNN_ERR_BITS;
    if (enc < 0 || enc > 3) return APNN_ERR_ENCODING;
    const bool apm = enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1;
    if (apm && a_bits != 1) return APNN_ERR_ENCODING;
    if (M > 0 && K > 0 && (!A || !Ap)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(Ap)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    // the int8 operand rows of apnn_prepare_weights_i8, with the +-1 decision taken on A's side
    cudaError_t err = launch_prepare_weights_i8(A, M, K, a_bits, apm ? APNN_ENC_PM1_PM1 : APNN_ENC_01_01, Ap, d.sms,
                                                (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_gemm_prepared_ab_i8(const uint8_t* Ap, const uint8_t* Wp, int M, int N, int K, int a_bits,
                                     int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                                     apnn_stream_t stream) {
    if (M < 0 || N < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if ((st = check_overflow(K, a_bits, w_bits, enc)) != APNN_OK) return st;  // int32 accumulators (R8)
    if ((M > 0 && K > 0 && !Ap) || (N > 0 && K > 0 && !Wp) || (M > 0 && N > 0 && !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(Ap) || !aligned16(Wp) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if (e.pool || e.res) return APNN_ERR_INVALID_ARG;
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (M == 0 || N == 0) return APNN_OK;
    cudaError_t err = launch_tc_i8_prepared_ab(Ap, Wp, g, e, Y, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

size_t apnn_prepared_i8_bytes(int N, int K) {
    if (N < 0 || K < 0) return 0;
    return (size_t)N * (((size_t)K + 127) / 128 * 128);
}

apnn_status apnn_prepare_weights_i8(const uint32_t* W, int N, int K, int w_bits, apnn_encoding enc, uint8_t* Wp,
                                    apnn_stream_t stream) {
    if (N < 0 || K < 0) return APNN_ERR_SHAPE;
    if (w_bits < 1 || w_bits > 8) return APNN_ERR_BITS;
    if (enc < 0 || enc > 3) return APNN_ERR_ENCODING;
    if ((enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_PM1_A_01) && w_bits != 1) return APNN_ERR_ENCODING;
    if (N > 0 && K > 0 && (!W || !Wp)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(W) || !aligned16(Wp)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st = device_info(&d);
    if (st != APNN_OK) return st;
    cudaError_t err = launch_prepare_weights_i8(W, N, K, w_bits, enc, Wp, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_gemm_prepared_i8(const uint32_t* A, const uint8_t* Wp, int M, int N, int K, int a_bits,
                                  int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                                  apnn_stream_t stream) {
    if (M < 0 || N < 0 || K < 0) return APNN_ERR_SHAPE;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if ((M > 0 && K > 0 && !A) || (N > 0 && K > 0 && !Wp) || (M > 0 && N > 0 && !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(Wp) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    if ((st = check_overflow(K, a_bits, w_bits, enc)) != APNN_OK) return st;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if (e.pool || e.res || M <= 128 || K == 0) return APNN_ERR_UNSUPPORTED;
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (N == 0) return APNN_OK;
    cudaError_t err = launch_tc_i8_prepared(A, Wp, g, e, Y, d.sms, (cudaStream_t)stream);
    if (err == cudaErrorNotSupported) return APNN_ERR_UNSUPPORTED;
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_tune_tiles(int M, int N, int K, int out_bits, int threshold, apnn_tile_config* out) {
    if (M < 1 || N < 1 || K < 1) return APNN_ERR_SHAPE;
    if (!out) return APNN_ERR_INVALID_ARG;
    const int T = threshold > 0 ? threshold : 64;  // the paper's T
    const TileCfg c = tune_tiles(M, N, K, T, out_bits > 0);
    out->kernel = c.kernel;
    out->bm = c.bm;
    out->bn = c.bn;
    out->ksplit = c.z;
    out->tlp = c.tlp;
    out->ci = c.ci;
    return APNN_OK;
}

apnn_status apnn_gemm_tiled(const uint32_t* A, const uint32_t* W, int M, int N, int K, int a_bits, int w_bits,
                            apnn_encoding enc, const apnn_epilogue* epi, void* Y, const apnn_tile_config* cfg,
                            apnn_stream_t stream) {
    if (M < 0 || N < 0 || K < 0) return APNN_ERR_SHAPE;
    if (!cfg) return APNN_ERR_INVALID_ARG;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if ((M > 0 && K > 0 && !A) || (N > 0 && K > 0 && !W) || (M > 0 && N > 0 && !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(W) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    if ((st = check_overflow(K, a_bits, w_bits, enc)) != APNN_OK) return st;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if (e.pool || e.res) return APNN_ERR_INVALID_ARG;
    const TileCfg c{cfg->kernel, cfg->bm, cfg->bn, cfg->ksplit, 0, 0.0};
    if (K == 0 || !tile_cfg_valid(c, M, N, K, e.out_bits > 0)) return APNN_ERR_UNSUPPORTED;
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (M == 0 || N == 0) return APNN_OK;
    cudaError_t err = launch_tc_i8_tiled(A, W, g, e, Y, c, d.sms, (cudaStream_t)stream);
    if (err == cudaErrorNotSupported) return APNN_ERR_UNSUPPORTED;
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_gemm(const uint32_t* A, const uint32_t* W, int M, int N, int K, int a_bits,
                      int w_bits, apnn_encoding enc, int32_t* Y, apnn_stream_t stream) {
    return apnn_gemm_ex(A, W, M, N, K, a_bits, w_bits, enc, nullptr, Y, APNN_VARIANT_AUTO, stream);
}

apnn_status apnn_gemm_fused(const uint32_t* A, const uint32_t* W, int M, int N, int K, int a_bits,
                            int w_bits, apnn_encoding enc, const apnn_epilogue* epi,
                            uint32_t* Y_packed, apnn_stream_t stream) {
    if (!epi) return APNN_ERR_INVALID_ARG;
    return apnn_gemm_ex(A, W, M, N, K, a_bits, w_bits, enc, epi, Y_packed, APNN_VARIANT_AUTO, stream);
}

static apnn_status conv_impl(const uint32_t* X, const void* W, bool prepared, const apnn_conv_shape* shp,
                             int a_bits, int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                             apnn_variant variant, apnn_stream_t stream);

apnn_status apnn_conv2d_prepared_i8(const uint32_t* X, const uint8_t* Wp, const apnn_conv_shape* shp, int a_bits,
                                    int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                                    apnn_stream_t stream) {
    return conv_impl(X, Wp, true, shp, a_bits, w_bits, enc, epi, Y, APNN_VARIANT_TC_I8, stream);
}

apnn_status apnn_conv2d_ex(const uint32_t* X, const uint32_t* W, const apnn_conv_shape* shp,
                           int a_bits, int w_bits, apnn_encoding enc, const apnn_epilogue* epi,
                           void* Y, apnn_variant variant, apnn_stream_t stream) {
    return conv_impl(X, W, false, shp, a_bits, w_bits, enc, epi, Y, variant, stream);
}

static apnn_status conv_impl(const uint32_t* X, const void* Wv, bool prepared, const apnn_conv_shape* shp,
                             int a_bits, int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                             apnn_variant variant, apnn_stream_t stream) {
    const uint32_t* W = reinterpret_cast<const uint32_t*>(Wv);
    if (!shp) return APNN_ERR_INVALID_ARG;
    const apnn_conv_shape c = *shp;
    if (c.B < 0 || c.H < 1 || c.W < 1 || c.C_in < 1 || c.C_out < 1 || c.R < 1 || c.S < 1 ||
        c.stride < 1 || c.pad < 0)
        return APNN_ERR_SHAPE;
    const int Ho = (c.H + 2 * c.pad - c.R) / c.stride + 1;
    const int Wo = (c.W + 2 * c.pad - c.S) / c.stride + 1;
    if (c.H + 2 * c.pad < c.R || c.W + 2 * c.pad < c.S || Ho < 1 || Wo < 1) return APNN_ERR_SHAPE;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    const long long Mll = (long long)c.B * Ho * Wo;
    const long long Kll = (long long)c.R * c.S * c.C_in;
    if (Mll > 2147483647LL || Kll > 2147483647LL) return APNN_ERR_SHAPE;
    if ((Mll > 0 && (!X || !W || !Y))) return APNN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(W) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    if ((st = check_overflow(Kll, a_bits, w_bits, enc)) != APNN_OK) return st;
    Epi e;
    if ((st = make_epi(epi, &e)) != APNN_OK) return st;
    if ((unsigned)variant > (unsigned)APNN_VARIANT_TC_FP4) return APNN_ERR_INVALID_ARG;
    Geom g;
    std::memset(&g, 0, sizeof(g));
    g.M = (int)Mll; g.N = c.C_out; g.K = (int)Kll;
    g.a_bits = a_bits; g.w_bits = w_bits; g.enc = enc;
    g.Cw = (c.C_in + 127) / 128 * 4;
    g.CB = g.Cw / 4;
    g.C = c.C_in;
    g.RS = c.R * c.S;
    g.nchunks = g.RS * g.CB;
    g.conv = 1;
    g.H = c.H; g.W = c.W; g.Ho = Ho; g.Wo = Wo; g.S = c.S; g.stride = c.stride; g.pad = c.pad;
    if (e.pool && (e.pool > Ho || e.pool > Wo)) return APNN_ERR_SHAPE;
    if (prepared && !(e.res && (enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1)) && conv_halo_enabled() &&
        conv_halo_supports(g, e)) {
        // tap-reuse kernel (conv_halo.cu): one decode per tile and channel chunk for all R*S taps
        DevInfo d;
        if ((st = device_info(&d)) != APNN_OK) return st;
        if (g.M == 0) return APNN_OK;
        cudaError_t err = launch_conv_halo(X, reinterpret_cast<const uint8_t*>(Wv), g, e, Y, d.sms,
                                           (cudaStream_t)stream);
        if (err == cudaErrorNotSupported) return APNN_ERR_UNSUPPORTED;
        return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
    }
    if (e.res && (resolve(variant, g, &e) != APNN_VARIANT_TC_I8 || g.M <= 128 || enc == APNN_ENC_PM1_PM1 ||
                  enc == APNN_ENC_W_01_A_PM1))
        return APNN_ERR_UNSUPPORTED;
    if (e.pool) {
        if (resolve(variant, g) != APNN_VARIANT_TC_I8 || !tc_i8_pool_fusable(g, e)) return APNN_ERR_UNSUPPORTED;
    }
    if (prepared) {
        if (g.M <= 128 || e.res) return APNN_ERR_UNSUPPORTED;
        DevInfo d;
        if ((st = device_info(&d)) != APNN_OK) return st;
        if (g.M == 0) return APNN_OK;
        cudaError_t err = launch_tc_i8_prepared(X, reinterpret_cast<const uint8_t*>(Wv), g, e, Y, d.sms,
                                                (cudaStream_t)stream);
        if (err == cudaErrorNotSupported) return APNN_ERR_UNSUPPORTED;
        return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
    }
    return run(X, W, g, e, Y, variant, (cudaStream_t)stream);
}

int apnn_conv_halo_fits(const apnn_conv_shape* shp, int a_bits, int w_bits, apnn_encoding enc,
                        const apnn_epilogue* epi) {
    if (!shp || check_bits_enc(a_bits, w_bits, enc) != APNN_OK) return 0;
    const apnn_conv_shape c = *shp;
    if (c.B < 1 || c.H < 1 || c.W < 1 || c.C_in < 1 || c.C_out < 1 || c.R < 1 || c.S < 1 || c.stride < 1 ||
        c.pad < 0 || c.H + 2 * c.pad < c.R || c.W + 2 * c.pad < c.S)
        return 0;
    Epi e;
    if (make_epi(epi, &e) != APNN_OK) return 0;
    if (e.res && (enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1)) return 0;
    Geom g;
    std::memset(&g, 0, sizeof(g));
    g.Ho = (c.H + 2 * c.pad - c.R) / c.stride + 1;
    g.Wo = (c.W + 2 * c.pad - c.S) / c.stride + 1;
    const long long Mll = (long long)c.B * g.Ho * g.Wo, Kll = (long long)c.R * c.S * c.C_in;
    if (Mll > 2147483647LL || Kll > 2147483647LL) return 0;
    g.M = (int)Mll; g.N = c.C_out; g.K = (int)Kll;
    g.a_bits = a_bits; g.w_bits = w_bits; g.enc = enc;
    g.Cw = (c.C_in + 127) / 128 * 4;
    g.CB = g.Cw / 4;
    g.C = c.C_in;
    g.RS = c.R * c.S;
    g.nchunks = g.RS * g.CB;
    g.conv = 1;
    g.H = c.H; g.W = c.W; g.S = c.S; g.stride = c.stride; g.pad = c.pad;
    return conv_halo_enabled() && conv_halo_supports(g, e) ? 1 : 0;
}

// First layer (raw 8-bit image, quantised inside the conv kernel): geometry of the contraction
// over taps r with K = the S x C_in window of one input row
static apnn_status first_geom(const apnn_conv_shape* shp, int zero_point, int scale, int a_bits, int w_bits,
                              apnn_encoding enc, const apnn_epilogue* epi, Geom* g, Epi* e) {
    if (!shp) return APNN_ERR_INVALID_ARG;
    const apnn_conv_shape c = *shp;
    if (c.B < 0 || c.H < 1 || c.W < 1 || c.C_in < 1 || c.C_out < 1 || c.R < 1 || c.S < 1 || c.stride < 1 ||
        c.pad < 0 || c.H + 2 * c.pad < c.R || c.W + 2 * c.pad < c.S)
        return APNN_ERR_SHAPE;
    if (scale < 1 || scale > 255 || zero_point < -255 || zero_point > 255) return APNN_ERR_INVALID_ARG;
    apnn_status st = check_bits_enc(a_bits, w_bits, enc);
    if (st != APNN_OK) return st;
    if (enc == APNN_ENC_PM1_PM1 || enc == APNN_ENC_W_01_A_PM1) return APNN_ERR_ENCODING;  // codes are 0/1 values
    if ((long long)c.S * c.C_in > 128) return APNN_ERR_UNSUPPORTED;                        // one copy row per window
    const int Ho = (c.H + 2 * c.pad - c.R) / c.stride + 1, Wo = (c.W + 2 * c.pad - c.S) / c.stride + 1;
    const long long Mll = (long long)c.B * Ho * Wo, Kll = (long long)c.R * c.S * c.C_in;
    if (Mll > 2147483647LL) return APNN_ERR_SHAPE;
    if ((st = check_overflow(Kll, a_bits, w_bits, enc)) != APNN_OK) return st;
    if ((st = make_epi(epi, e)) != APNN_OK) return st;
    if (e->res) return APNN_ERR_UNSUPPORTED;
    std::memset(g, 0, sizeof(*g));
    g->M = (int)Mll; g->N = c.C_out; g->K = (int)Kll;
    g->a_bits = a_bits; g->w_bits = w_bits; g->enc = enc;
    g->C = c.S * c.C_in;  // virtual channels: the window
    g->Cw = 4;
    g->CB = 1;
    g->RS = c.R;          // taps: rows
    g->nchunks = c.R;
    g->conv = 1;
    g->H = c.H; g->W = c.W; g->Ho = Ho; g->Wo = Wo; g->S = 1; g->stride = c.stride; g->pad = c.pad;
    return APNN_OK;
}

int apnn_conv_first_fits(const apnn_conv_shape* shp, int a_bits, int w_bits, apnn_encoding enc,
                         const apnn_epilogue* epi) {
    Geom g;
    Epi e;
    if (first_geom(shp, 0, 1, a_bits, w_bits, enc, epi, &g, &e) != APNN_OK) return 0;
    return conv_first_supports(g, e, shp->S, shp->C_in) ? 1 : 0;
}

apnn_status apnn_conv2d_first_prepared_i8(const uint8_t* X, const uint8_t* Wp, const apnn_conv_shape* shp,
                                          int zero_point, int scale, int a_bits, int w_bits, apnn_encoding enc,
                                          const apnn_epilogue* epi, void* Y, apnn_stream_t stream) {
    Geom g;
    Epi e;
    apnn_status st = first_geom(shp, zero_point, scale, a_bits, w_bits, enc, epi, &g, &e);
    if (st != APNN_OK) return st;
    if (g.M > 0 && (!X || !Wp || !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(Wp) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    if (e.pool && (e.pool > g.Ho || e.pool > g.Wo)) return APNN_ERR_SHAPE;
    if (!conv_first_supports(g, e, shp->S, shp->C_in)) return APNN_ERR_UNSUPPORTED;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (g.M == 0) return APNN_OK;
    cudaError_t err = launch_conv_first(X, Wp, g, e, zero_point, scale, shp->S, shp->C_in, Y, d.sms,
                                        (cudaStream_t)stream);
    if (err == cudaErrorNotSupported) return APNN_ERR_UNSUPPORTED;
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_conv2d(const uint32_t* X, const uint32_t* W, const apnn_conv_shape* shp, int a_bits,
                        int w_bits, apnn_encoding enc, const apnn_epilogue* epi, void* Y,
                        apnn_stream_t stream) {
    return apnn_conv2d_ex(X, W, shp, a_bits, w_bits, enc, epi, Y, APNN_VARIANT_AUTO, stream);
}

apnn_status apnn_quant_pack_out(const int32_t* Y, int M, int N, const apnn_epilogue* epi,
                                uint32_t* out, apnn_stream_t stream) {
    if (M < 0 || N < 0) return APNN_ERR_SHAPE;
    if (!epi) return APNN_ERR_INVALID_ARG;
    if ((M > 0 && N > 0 && !Y) || (M > 0 && !out)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(Y) || !aligned16(out)) return APNN_ERR_ALIGNMENT;
    Epi e;
    apnn_status st = make_epi(epi, &e);
    if (st != APNN_OK) return st;
    if (e.pool) return APNN_ERR_INVALID_ARG;  // pooled: apnn_pool_quant_pack_out
    if (e.res) return APNN_ERR_INVALID_ARG;  // residual: apnn_residual_quant_pack
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    cudaError_t err = launch_quant_pack(Y, M, N, e, out, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_pool_quant_pack_out(const int32_t* Y, int B, int H, int W, int N, const apnn_epilogue* epi,
                                     uint32_t* out, apnn_stream_t stream) {
    if (B < 0 || H < 1 || W < 1 || N < 0) return APNN_ERR_SHAPE;
    if (!epi) return APNN_ERR_INVALID_ARG;
    Epi e;
    apnn_status st = make_epi(epi, &e);
    if (st != APNN_OK) return st;
    if (e.pool < 1 || e.res) return APNN_ERR_INVALID_ARG;
    if (e.pool > H || e.pool > W) return APNN_ERR_SHAPE;
    const int Hp = (H - e.pool) / e.pool_stride + 1, Wp = (W - e.pool) / e.pool_stride + 1;
    if ((long long)B * Hp * Wp > 2147483647LL) return APNN_ERR_SHAPE;
    if ((B > 0 && N > 0 && !Y) || (B > 0 && !out)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(Y) || !aligned16(out)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    cudaError_t err = launch_pool_quant_pack(Y, B, H, W, N, e, out, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_maxpool_packed(const uint32_t* X, int B, int H, int W, int C, int bits, int k, int stride,
                                uint32_t* Y, apnn_stream_t stream) {
    if (B < 0 || H < 1 || W < 1 || C < 0) return APNN_ERR_SHAPE;
    if (bits < 1 || bits > 8) return APNN_ERR_BITS;
    if (k < 1 || stride < 1) return APNN_ERR_INVALID_ARG;
    if (k > H || k > W) return APNN_ERR_SHAPE;
    const int Hp = (H - k) / stride + 1, Wp = (W - k) / stride + 1;
    if ((long long)B * H * W > 2147483647LL || (long long)B * Hp * Wp > 2147483647LL) return APNN_ERR_SHAPE;
    if (B > 0 && C > 0 && (!X || !Y)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(Y)) return APNN_ERR_ALIGNMENT;
    DevInfo d;
    apnn_status st;
    if ((st = device_info(&d)) != APNN_OK) return st;
    if (B == 0 || C == 0) return APNN_OK;
    cudaError_t err = launch_maxpool_packed(X, B, H, W, C, bits, k, stride, Y, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_status apnn_residual_quant_pack(const int32_t* Y, int M, int N, const void* Z, int z_bits,
                                     const int32_t* rho, const apnn_epilogue* epi, uint32_t* out,
                                     apnn_stream_t stream) {
    if (M < 0 || N < 0) return APNN_ERR_SHAPE;
    if (!epi) return APNN_ERR_INVALID_ARG;
    if (z_bits < 0 || z_bits > 8) return APNN_ERR_BITS;
    if ((M > 0 && N > 0 && (!Y || !Z)) || (M > 0 && !out)) return APNN_ERR_INVALID_ARG;
    if (!aligned16(Y) || !aligned16(Z) || !aligned16(out) || (rho && !aligned16(rho))) return APNN_ERR_ALIGNMENT;
    Epi e;
    apnn_status st = make_epi(epi, &e);
    if (st != APNN_OK) return st;
    if (e.pool || e.res) return APNN_ERR_INVALID_ARG;  // the shortcut is the Z argument here
    DevInfo d;
    if ((st = device_info(&d)) != APNN_OK) return st;
    cudaError_t err = launch_residual_quant_pack(Y, M, N, Z, z_bits, rho, e, out, d.sms, (cudaStream_t)stream);
    return err == cudaSuccess ? APNN_OK : APNN_ERR_CUDA;
}

apnn_variant apnn_select_variant(int M, int N, int K, int a_bits, int w_bits, apnn_encoding enc) {
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    return resolve(APNN_VARIANT_AUTO, g);
}

apnn_variant apnn_select_variant_fused(int M, int N, int K, int a_bits, int w_bits, apnn_encoding enc,
                                       int out_bits) {
    Geom g;
    gemm_geom(&g, M, N, K, a_bits, w_bits, enc);
    Epi e;
    std::memset(&e, 0, sizeof(e));
    e.out_bits = out_bits;
    return resolve(APNN_VARIANT_AUTO, g, &e);
}

const char* apnn_status_string(apnn_status s) {
    switch (s) {
    case APNN_OK: return "ok";
    case APNN_ERR_INVALID_ARG: return "invalid argument";
    case APNN_ERR_BITS: return "bit width outside 1..8";
    case APNN_ERR_ENCODING: return "illegal encoding for these bit widths";
    case APNN_ERR_SHAPE: return "bad shape";
    case APNN_ERR_ALIGNMENT: return "device pointer not 16-byte aligned";
    case APNN_ERR_OVERFLOW: return "worst-case result exceeds int32";
    case APNN_ERR_UNSUPPORTED: return "unsupported by the requested kernel variant";
    case APNN_ERR_CUDA: return "CUDA error (no sm_100 device or launch failure)";
    }
    return "unknown status";
}

const char* apnn_variant_name(apnn_variant v) {
    switch (v) {
    case APNN_VARIANT_AUTO: return "auto";
    case APNN_VARIANT_TC_I8: return "tc_i8";
    case APNN_VARIANT_POPC: return "popc";
    case APNN_VARIANT_B1MMA: return "b1mma";
    case APNN_VARIANT_TC_FP4: return "tc_fp4";
    }
    return "unknown";
}

uint64_t apnn_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int apnn_version(void) { return 300; }  // 0.3.0: both-prepared GEMMs, fused / dense decomposition, packed max pool

}  // extern "C"
