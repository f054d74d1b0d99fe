// streaming.cu -- HBM-bound element-wise kernels of the AP-bit path.
//
//   pack_bits_kernel      bit decomposition + packing (Eq. bitDecomposition,
//                         PAPER.md:1419-1421) of uint8 codes into the packed
//                         bit-plane format of include/apnn.h.
//   quant_pack_kernel     the stand-alone element-wise routine: requantise int32
//                         and re-pack; the unfused
//                         counterpart of the GEMM epilogue.
//
// One thread produces one 32-bit word per plane (32 codes).  Loads are 128-bit
// and contiguous per thread, stores of consecutive threads are consecutive
// words of one plane run -> both sides coalesce.  Grids are sized in multiples
// of the SM count by the launcher (grid-stride loops).
#include <cstdlib>

#include "common.cuh"

namespace apnn {

// codes [rows][K] -> dst [rows][bits][Kw].  PREP (apnn_pack_bits_prepared, <= 2-bit codes): the
// same thread also writes the 32 codes' e2m1 operand bytes (the rows of apnn_prepare_activations:
// word j of a 32-element group holds elements j, j+4, ..., j+28; 0/1 codes v -> value v, +-1
// codes (PM1) -> +-1.0 with elements >= K value 0), so the GEMM's A operand comes out of the bit
// decomposition without a second pass over the planes.  x over a row's words, y over rows,
// 32-bit index math.
template <bool kVec, bool PREP, bool PM1>
__global__ void __launch_bounds__(256) pack_bits_kernel(const uint8_t* __restrict__ codes, int rows,
                                                        int K, int bits, int Kw,
                                                        uint32_t* __restrict__ dst, uint8_t* __restrict__ prep) {
    const uint32_t keep = (bits >= 8) ? 0xFFFFFFFFu : (0x01010101u * ((1u << bits) - 1u));
    for (int r = blockIdx.y * blockDim.y + threadIdx.y; r < rows; r += gridDim.y * blockDim.y) {
        const uint8_t* crow = codes + (long long)r * K;
        uint32_t* out = dst + (long long)r * bits * Kw;
        for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < Kw; w += gridDim.x * blockDim.x) {
            const int k0 = w * 32;
            uint32_t u[8];
            if (k0 + 32 <= K) {
                const uint8_t* src = crow + k0;
                if (kVec) {
                    uint4 v0 = __ldg(reinterpret_cast<const uint4*>(src));
                    uint4 v1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
                    u[0] = v0.x; u[1] = v0.y; u[2] = v0.z; u[3] = v0.w;
                    u[4] = v1.x; u[5] = v1.y; u[6] = v1.z; u[7] = v1.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        u[q] = (uint32_t)src[4 * q] | ((uint32_t)src[4 * q + 1] << 8) |
                               ((uint32_t)src[4 * q + 2] << 16) | ((uint32_t)src[4 * q + 3] << 24);
                }
            } else {
                // ragged tail / padding run: codes beyond K are zero
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    uint32_t x = 0;
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        int k = k0 + 4 * q + b;
                        if (k < K) x |= (uint32_t)crow[k] << (8 * b);
                    }
                    u[q] = x;
                }
            }
#pragma unroll
            for (int q = 0; q < 8; q++) u[q] &= keep;  // codes are masked to their low `bits` bits
            uint32_t pw[2] = {0u, 0u};
            for (int t = 0; t < bits; t++) {
                uint32_t word = 0;
#pragma unroll
                for (int q = 0; q < 8; q++) word |= byte_bits_to_nibble(u[q], t) << (4 * q);
                out[(long long)t * Kw + w] = word;
                if (PREP && t < 2) pw[t] = word;
            }
            if (PREP) {
                const int nv = K - k0;
                const uint32_t vm = nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
                uint32_t o[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint32_t b0 = (pw[0] >> j) & 0x11111111u, b1 = (pw[1] >> j) & 0x11111111u;
                    uint32_t v;
                    if (PM1) v = 0x22222222u | ((b0 ^ 0x11111111u) << 3);  // +1 -> 0x2, -1 -> 0xA
                    else v = (b1 << 2) | ((b0 & ~b1) << 1) | (b0 & b1);    // 0..3 -> 0x0, 0x2, 0x4, 0x5
                    o[j] = v & (((vm >> j) & 0x11111111u) * 0xFu);         // elements >= K: value 0
                }
                *reinterpret_cast<uint4*>(prep + ((long long)r * Kw + w) * 16) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// The element-wise routines (unfused forms of the epilogue):
//   quant_pack      q = requant(alpha*y + beta)                      (apnn_quant_pack_out)
//   pool_quant_pack q = requant(pool_kxk(alpha*y + beta))            (R15)
//   residual        q = requant(alpha*y + beta + rho*z)              (reading R24)
// all writing packed planes [rows][ob][Nw].  Work split: a warp owns ONE output word column
// w (32 consecutive channels, lane = channel: coalesced 128-byte loads of int32 rows) and
// walks the rows r0, r0 + rstride, ... (kRows of them in flight), so the per-channel
// parameters are loaded once per warp; each plane word is one __ballot_sync (the paper's
// ballot packing).  Only words that hold channels are walked; the
// warp of the last one also writes the row's zero padding words.  The host sizes the grid
// so that the number of warps is a multiple of the word count.
constexpr int kRows = 4;

struct WordWalk {
    int w, r0, rstride;
};
__device__ __forceinline__ WordWalk word_walk(int Nd) {
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    return WordWalk{gw % Nd, gw / Nd, nwarps / Nd};
}

// Requantisation constants of one launch: q = clamp(floor(v / S), 0, qmax) of an int64 v.
struct QuantK {
    long long lim;  // (qmax + 1) * S: v >= lim -> qmax
    uint32_t S, qmax;
    float invS;
};
static QuantK quant_k(const Epi& e) {
    return QuantK{(long long)(e.qmax + 1) * e.S, (uint32_t)e.S, (uint32_t)e.qmax, e.invS};
}
// FAST (host: lim <= 2^32): the in-range v fits 32 bits and an fp32 estimate is within one
// of the floor (relative error < 2^-22 on q <= 255), fixed by one exact integer correction.
template <bool FAST>
__device__ __forceinline__ uint32_t quant_v(long long v, const QuantK& k, const Epi& e) {
    if (v < 0) return 0u;
    if (v >= k.lim) return k.qmax;
    if (!FAST) return quantise_v(e, v);
    const uint32_t u = (uint32_t)v;
    uint32_t q = __float2uint_rz(__uint2float_rn(u) * k.invS);
    const int32_t r = (int32_t)(u - q * k.S);
    return r < 0 ? q - 1 : (r >= (int32_t)k.S ? q + 1 : q);
}

// planes of 32 lanes' codes -> lane t < ob stores plane t's word of this row; with
// pad_words > 0 (the row's last data word) lanes also zero the words w+1 .. w+pad_words
template <int OB>
__device__ __forceinline__ void ballot_store(uint32_t q, int lane, int ob, uint32_t* row_words, int Nw,
                                             int pad_words) {
    const int nb = OB > 0 ? OB : ob;
    uint32_t mine = 0;
#pragma unroll
    for (int t = 0; t < 8; t++) {
        if (t < nb) {
            const uint32_t word = __ballot_sync(0xFFFFFFFFu, (q >> t) & 1u);
            if (lane == t) mine = word;
        }
    }
    if (lane < nb) row_words[(long long)lane * Nw] = mine;
    for (int i = lane; i < pad_words * nb; i += 32) row_words[(long long)(i / pad_words) * Nw + 1 + i % pad_words] = 0u;
}

template <bool FAST, int OB>
__global__ void __launch_bounds__(256) quant_pack_kernel(const int32_t* __restrict__ Y, int M, int N, int Nd,
                                                         int Nw, Epi e, QuantK qk, uint32_t* __restrict__ out) {
    const WordWalk k = word_walk(Nd);
    const int lane = threadIdx.x & 31, n = k.w * 32 + lane, ob = OB > 0 ? OB : e.out_bits;
    const bool valid = n < N;
    const int32_t al = valid ? epi_alpha(e, n) : 0, be = valid ? epi_beta(e, n) : 0;
    const int pad = k.w == Nd - 1 ? Nw - Nd : 0;
    for (int r = k.r0; r < M; r += kRows * k.rstride) {
        int32_t y[kRows];
#pragma unroll
        for (int u = 0; u < kRows; u++) {
            const int row = r + u * k.rstride;
            y[u] = (valid && row < M) ? __ldg(Y + (long long)row * N + n) : 0;
        }
#pragma unroll
        for (int u = 0; u < kRows; u++) {
            const int row = r + u * k.rstride;
            if (row >= M) break;  // warp-uniform
            const uint32_t q = valid ? quant_v<FAST>((long long)al * y[u] + be, qk, e) : 0u;
            ballot_store<OB>(q, lane, ob, out + (long long)row * ob * Nw + k.w, Nw, pad);
        }
    }
}

// Y [B][H][W][N] (NHWC conv output) -> pooled rows [B*Hp*Wp].  Max pooling of v = alpha*y + beta
// is alpha*max(y) + beta for alpha >= 0 and alpha*min(y) + beta otherwise (v is monotone in y):
// the window is reduced in 32-bit and v is formed once per output.  Average: floor of
// (alpha*sum(y) + k*k*beta) / (k*k) (reading R15).
template <int KP, bool FAST, int OB>
__global__ void __launch_bounds__(256) pool_quant_pack_kernel(const int32_t* __restrict__ Y, int B, int H, int W,
                                                              int N, int Hp, int Wp, int Nd, int Nw, Epi e,
                                                              QuantK qk, uint32_t* __restrict__ out) {
    const WordWalk k = word_walk(Nd);
    const int lane = threadIdx.x & 31, n = k.w * 32 + lane, ob = OB > 0 ? OB : e.out_bits;
    const bool valid = n < N;
    const int32_t al = valid ? epi_alpha(e, n) : 0, be = valid ? epi_beta(e, n) : 0;
    const int kp = KP > 0 ? KP : e.pool, st = e.pool_stride;
    const int pad = k.w == Nd - 1 ? Nw - Nd : 0;
    const int P = B * Hp * Wp;
    const bool avg = e.pool_avg != 0;
    for (int r = k.r0; r < P; r += kRows * k.rstride) {
        int32_t ysel[kRows];  // max (alpha >= 0) or min (alpha < 0) of the window
        long long ysum[kRows];
#pragma unroll
        for (int u = 0; u < kRows; u++) {
            const int pix = r + u * k.rstride;
            ysel[u] = 0;
            ysum[u] = 0;
            if (valid && pix < P) {
                const int b = pix / (Hp * Wp), rem = pix - b * Hp * Wp;
                const int i = rem / Wp, j = rem - (rem / Wp) * Wp;
                const int32_t* base = Y + (((long long)b * H + i * st) * W + j * st) * N + n;
                int32_t mx = INT32_MIN, mn = INT32_MAX;
                long long sm = 0;
#pragma unroll
                for (int rr = 0; rr < kp; rr++) {  // kp is the constant KP in the KP > 0 instances
#pragma unroll
                    for (int ss = 0; ss < kp; ss++) {
                        const int32_t yv = __ldg(base + ((long long)rr * W + ss) * N);
                        mx = max(mx, yv);
                        mn = min(mn, yv);
                        if (avg) sm += yv;
                    }
                }
                ysel[u] = al >= 0 ? mx : mn;
                ysum[u] = sm;
            }
        }
#pragma unroll
        for (int u = 0; u < kRows; u++) {
            const int pix = r + u * k.rstride;
            if (pix >= P) break;  // warp-uniform
            uint32_t q = 0;
            if (valid) {
                long long v;
                if (avg) {
                    const long long kk = (long long)kp * kp, t = (long long)al * ysum[u] + kk * be;
                    v = t / kk;
                    if (t % kk != 0 && t < 0) v -= 1;  // floor toward -inf
                } else {
                    v = (long long)al * ysel[u] + be;
                }
                q = quant_v<FAST>(v, qk, e);
            }
            ballot_store<OB>(q, lane, ob, out + (long long)pix * ob * Nw + k.w, Nw, pad);
        }
    }
}

// shortcut z: int32 [M][N] (ZB = 0) or packed codes [M][z_bits][Nw] (ZB = -1: runtime z_bits)
template <bool FAST, int OB, int ZB>
__global__ void __launch_bounds__(256) residual_quant_pack_kernel(const int32_t* __restrict__ Y, int M, int N,
                                                                  const void* __restrict__ Z, int z_bits,
                                                                  const int32_t* __restrict__ rho, int Nd, int Nw,
                                                                  Epi e, QuantK qk, uint32_t* __restrict__ out) {
    const WordWalk k = word_walk(Nd);
    const int lane = threadIdx.x & 31, n = k.w * 32 + lane, ob = OB > 0 ? OB : e.out_bits;
    const bool valid = n < N;
    const int32_t al = valid ? epi_alpha(e, n) : 0, be = valid ? epi_beta(e, n) : 0;
    const int32_t rh = valid ? (rho ? __ldg(rho + n) : 1) : 0;
    const int pad = k.w == Nd - 1 ? Nw - Nd : 0;
    const int32_t* Zi = reinterpret_cast<const int32_t*>(Z);
    const uint32_t* Zp = reinterpret_cast<const uint32_t*>(Z);
    for (int r = k.r0; r < M; r += kRows * k.rstride) {
        int32_t y[kRows];
        uint32_t zw[kRows];  // ZB != 0: lane t < z_bits holds plane t's word of the row
        int32_t zi[kRows];
#pragma unroll
        for (int u = 0; u < kRows; u++) {
            const int row = r + u * k.rstride;
            y[u] = zi[u] = 0;
            zw[u] = 0;
            if (row < M) {
                if (valid) y[u] = __ldg(Y + (long long)row * N + n);
                if (ZB == 0) {
                    if (valid) zi[u] = __ldg(Zi + (long long)row * N + n);
                } else if (lane < z_bits) {
                    zw[u] = __ldg(Zp + ((long long)row * z_bits + lane) * Nw + k.w);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kRows; u++) {
            const int row = r + u * k.rstride;
            if (row >= M) break;  // warp-uniform
            int32_t z = zi[u];
            if (ZB != 0) {  // this lane's code: bit `lane` of every plane word (shuffled from lane t)
                uint32_t code = 0;
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    if (t < z_bits) code |= ((__shfl_sync(0xFFFFFFFFu, zw[u], t) >> lane) & 1u) << t;
                }
                z = (int32_t)code;
            }
            const uint32_t q = valid ? quant_v<FAST>((long long)al * y[u] + be + (long long)rh * z, qk, e) : 0u;
            ballot_store<OB>(q, lane, ob, out + (long long)row * ob * Nw + k.w, Nw, pad);
        }
    }
}

static int stream_grid(long long total, int sms) {
    long long blocks = (total + 255) / 256;
    long long cap = (long long)sms * 8;  // 8 resident 256-thread CTAs per SM, grid-stride beyond
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

// grid for the word-walk routines: enough warps to cover rows x Nd (capped at 8 CTAs per SM),
// rounded up to a multiple of Nd CTAs so the warp count is a multiple of Nd
static int word_grid(long long rows, int Nd, int sms) {
    long long blocks = (rows * Nd + 7) / 8;
    const long long cap = (long long)sms * 8;
    if (blocks > cap) blocks = cap;
    blocks = (blocks + Nd - 1) / Nd * Nd;
    return (int)(blocks < Nd ? Nd : blocks);
}

static bool quant_fast(const Epi& e) {
    return (unsigned long long)(e.qmax + 1) * (unsigned long long)e.S <= 0x100000000ull;
}

cudaError_t launch_quant_pack(const int32_t* Y, int M, int N, const Epi& e, uint32_t* out, int sms,
                              cudaStream_t s) {
    const int Nw = (N + 127) / 128 * 4, Nd = (N + 31) / 32;
    if ((long long)M * Nw == 0) return cudaSuccess;
    const int grid = word_grid(M, Nd, sms);
    const QuantK qk = quant_k(e);
#define APNN_QP(F_, OB_) quant_pack_kernel<F_, OB_><<<grid, 256, 0, s>>>(Y, M, N, Nd, Nw, e, qk, out)
    if (!quant_fast(e)) APNN_QP(false, 0);
    else if (e.out_bits == 2) APNN_QP(true, 2);
    else if (e.out_bits == 8) APNN_QP(true, 8);
    else APNN_QP(true, 0);
#undef APNN_QP
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pool_quant_pack(const int32_t* Y, int B, int H, int W, int N, const Epi& e, uint32_t* out,
                                  int sms, cudaStream_t s) {
    const int Hp = (H - e.pool) / e.pool_stride + 1, Wp = (W - e.pool) / e.pool_stride + 1;
    const int Nw = (N + 127) / 128 * 4, Nd = (N + 31) / 32;
    const long long rows = (long long)B * Hp * Wp;
    if (rows * Nw == 0) return cudaSuccess;
    if (rows > 2147483647LL) return cudaErrorInvalidValue;
    const int grid = word_grid(rows, Nd, sms);
    const QuantK qk = quant_k(e);
    const bool f = quant_fast(e);
#define APNN_POOL(KP_, F_, OB_) \
    pool_quant_pack_kernel<KP_, F_, OB_><<<grid, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nd, Nw, e, qk, out)
    if (!f) APNN_POOL(0, false, 0);
    else if (e.pool == 2 && e.out_bits == 2) APNN_POOL(2, true, 2);
    else if (e.pool == 2 && e.out_bits == 8) APNN_POOL(2, true, 8);
    else if (e.pool == 3 && e.out_bits == 2) APNN_POOL(3, true, 2);
    else if (e.pool == 2) APNN_POOL(2, true, 0);
    else if (e.pool == 3) APNN_POOL(3, true, 0);
    else APNN_POOL(0, true, 0);
#undef APNN_POOL
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_residual_quant_pack(const int32_t* Y, int M, int N, const void* Z, int z_bits,
                                       const int32_t* rho, const Epi& e, uint32_t* out, int sms, cudaStream_t s) {
    const int Nw = (N + 127) / 128 * 4, Nd = (N + 31) / 32;
    if ((long long)M * Nw == 0) return cudaSuccess;
    const int grid = word_grid(M, Nd, sms);
    const QuantK qk = quant_k(e);
#define APNN_RES(F_, OB_, ZB_) \
    residual_quant_pack_kernel<F_, OB_, ZB_><<<grid, 256, 0, s>>>(Y, M, N, Z, z_bits, rho, Nd, Nw, e, qk, out)
    if (!quant_fast(e)) { if (z_bits) APNN_RES(false, 0, -1); else APNN_RES(false, 0, 0); }
    else if (e.out_bits == 8) { if (z_bits) APNN_RES(true, 8, -1); else APNN_RES(true, 8, 0); }
    else if (e.out_bits == 2) { if (z_bits) APNN_RES(true, 2, -1); else APNN_RES(true, 2, 0); }
    else { if (z_bits) APNN_RES(true, 0, -1); else APNN_RES(true, 0, 0); }
#undef APNN_RES
    count_launch();
    return cudaGetLastError();
}

// im2col + bit decomposition + packing of NHWC uint8 codes.  One CTA per output image
// row (b, ho): the R input rows it needs are staged in shared memory with the zero
// padding materialised (R x (W + 2 pad) x C bytes); qs > 0 quantises the raw 8-bit image
// while staging, q = clamp(floor((x - qz) / qs), 0, 2^bits - 1) (the first layer's
// quantisation of the 8-bit input, formula PAPER.md:1283-1287;
// out-of-frame taps stay code 0).  An offset table built once per CTA maps element
// k = (r*S + s)*C + c of a row to its staged byte for wo = 0 (k >= K -> a zero byte), so a
// task (pixel wo, word w) is 32 table-driven byte loads, then the plane words: shift-ors
// for <= 4 bits, 8x8 bit-matrix transposes above.  The CTA's Wo output rows are one
// contiguous range: words are staged in shared memory and written out coalesced.
__global__ void __launch_bounds__(256) im2col_pack_kernel(const uint8_t* __restrict__ X, int B, int H, int W,
                                                          int C, int R, int S, int stride, int pad, int Ho, int Wo,
                                                          int bits, int Kw, uint32_t* __restrict__ dst, int qz,
                                                          int qs) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int Wp = W + 2 * pad, rowb = Wp * C;       // padded input row bytes
    const int Kp = Kw * 32, K = R * S * C, SC = S * C;
    uint8_t* rows = sm;                              // R x rowb, then one zero byte
    const int zero_off = R * rowb;
    int32_t* tab = reinterpret_cast<int32_t*>(sm + ((R * rowb + 1 + 15) & ~15));            // Kp offsets
    uint32_t* outw = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(tab) + Kp * 4);   // Wo x bits x Kw
    const uint32_t keep = (1u << bits) - 1u;
    for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
        const int r = k / SC, j = k - r * SC;
        tab[k] = k < K ? r * rowb + j : -1;  // -1: the zero byte (wo-independent)
    }
    if (threadIdx.x == 0) rows[zero_off] = 0;
    for (int br = blockIdx.x; br < B * Ho; br += gridDim.x) {
        const int b = br / Ho, ho = br - b * Ho;
        __syncthreads();  // previous row's smem readers are done (and the table is built)
        for (int i = threadIdx.x; i < R * Wp; i += blockDim.x) {  // one padded pixel (C bytes) per step
            const int r = i / Wp, px = i - r * Wp;
            const int hi = ho * stride - pad + r, wi = px - pad;
            uint8_t* d = rows + r * rowb + px * C;
            if (hi >= 0 && hi < H && wi >= 0 && wi < W) {
                const uint8_t* src = X + (((long long)b * H + hi) * W + wi) * C;
                if (qs > 0) {
                    for (int c = 0; c < C; c++) {
                        const int v = (int)__ldg(src + c) - qz;  // floor((x - z) / s), clamped
                        const int q = v < 0 ? 0 : v / qs;
                        d[c] = (uint8_t)(q > (int)keep ? keep : q);
                    }
                } else {
                    for (int c = 0; c < C; c++) d[c] = __ldg(src + c) & keep;
                }
            } else {
                for (int c = 0; c < C; c++) d[c] = 0;
            }
        }
        __syncthreads();
        for (int task = threadIdx.x; task < Wo * Kw; task += blockDim.x) {
            const int wo = task / Kw, w = task - wo * Kw;
            const int base = wo * stride * C;
            const int4* t4 = reinterpret_cast<const int4*>(tab + w * 32);
            uint32_t qb[8];  // byte i of qb[j] = code of element 4j + i (as in pack_bits_kernel)
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int4 o = t4[j];
                const uint32_t c0 = rows[o.x < 0 ? zero_off : o.x + base];
                const uint32_t c1 = rows[o.y < 0 ? zero_off : o.y + base];
                const uint32_t c2 = rows[o.z < 0 ? zero_off : o.z + base];
                const uint32_t c3 = rows[o.w < 0 ? zero_off : o.w + base];
                qb[j] = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
            }
            uint32_t* o = outw + wo * bits * Kw + w;
            if (bits > 4) {  // 8x8 bit-matrix transposes: byte t of group g = plane t of codes 8g..8g+7
                uint32_t pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    unsigned long long x = ((unsigned long long)qb[2 * g + 1] << 32) | qb[2 * g];
                    unsigned long long d = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
                    x ^= d ^ (d << 7);
                    d = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
                    x ^= d ^ (d << 14);
                    d = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
                    x ^= d ^ (d << 28);
#pragma unroll
                    for (int t = 0; t < 8; t++) pw[t] |= (uint32_t)((x >> (8 * t)) & 0xFFull) << (8 * g);
                }
#pragma unroll
                for (int t = 0; t < 8; t++)
                    if (t < bits) o[t * Kw] = pw[t];
            } else {
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    if (t < bits) {
                        uint32_t word = 0;
#pragma unroll
                        for (int q = 0; q < 8; q++) word |= byte_bits_to_nibble(qb[q], t) << (4 * q);
                        o[t * Kw] = word;
                    }
                }
            }
        }
        __syncthreads();
        uint4* g = reinterpret_cast<uint4*>(dst + (long long)br * Wo * bits * Kw);  // rows (b, ho, 0..Wo-1)
        const uint4* sw = reinterpret_cast<const uint4*>(outw);                      // are contiguous
        for (int i = threadIdx.x; i < Wo * bits * Kw / 4; i += blockDim.x) g[i] = sw[i];
    }
}

// [B][P][bits][Cw] -> [B][bits][P*Cw] word permutation; thread = one destination word
__global__ void __launch_bounds__(256) flatten_packed_kernel(const uint32_t* __restrict__ src, int B, int P,
                                                             int bits, int Cw, uint32_t* __restrict__ dst) {
    const long long total = (long long)B * P * bits * Cw;
    const long long rowlen = (long long)P * Cw;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long b = idx / (bits * rowlen);
        long long r = idx - b * bits * rowlen;
        const int t = (int)(r / rowlen);
        r -= (long long)t * rowlen;
        const int pix = (int)(r / Cw), w = (int)(r - (long long)pix * Cw);
        dst[idx] = __ldg(src + (((b * P + pix) * bits + t) * Cw + w));
    }
}

// Dense codes (apnn_pack_bits_dense): `BITS`-bit codes stored back to back, LSB first, each row
// starting on a byte boundary (ceil(K * BITS / 8) bytes) -- the compact host format of low-bit
// activations.  A thread takes the 32 * BITS bits of one 32-element group; for BITS = 2 plane t is
// bit t of every 2-bit field, gathered by a 64 -> 32-bit compress; PREP writes the e2m1 rows too.
__device__ __forceinline__ uint32_t compress_even_bits(unsigned long long x) {
    x &= 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
    x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
    x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
    return (uint32_t)x;
}

template <int BITS, bool ALIGNED, bool PREP, bool PM1>
__device__ __forceinline__ unsigned long long dense_group(const uint8_t* crow, int k0, int K) {
    const int nv = K - k0;  // valid elements of this group
    unsigned long long x = 0;
    if (nv > 0) {
        const int b0 = k0 * BITS / 8, nb = BITS * 4;  // bytes of a full group
        if (ALIGNED && nv >= 32) {
            x = BITS == 2 ? __ldg(reinterpret_cast<const unsigned long long*>(crow + b0))
                          : (unsigned long long)__ldg(reinterpret_cast<const uint32_t*>(crow + b0));
        } else {
            const int have = (nv * BITS + 7) / 8 < nb ? (nv * BITS + 7) / 8 : nb;
            for (int i = 0; i < have; i++) x |= (unsigned long long)crow[b0 + i] << (8 * i);
        }
        if (nv < 32) x &= (BITS * nv >= 64) ? ~0ull : ((1ull << (BITS * nv)) - 1ull);
    }
    return x;
}

template <int BITS, bool ALIGNED, bool PREP, bool PM1>
__global__ void __launch_bounds__(256) pack_dense_kernel(const uint8_t* __restrict__ codes, int rows, int K,
                                                         int row_bytes, int Kw, uint32_t* __restrict__ dst,
                                                         uint8_t* __restrict__ prep) {
    constexpr int RU = 4;  // rows per pass: their loads are all in flight before any store
    const int rstep = gridDim.y * blockDim.y;
    for (int r0 = blockIdx.y * blockDim.y + threadIdx.y; r0 < rows; r0 += RU * rstep) {
        for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < Kw; w += gridDim.x * blockDim.x) {
            const int k0 = w * 32;
            unsigned long long x[RU];
#pragma unroll
            for (int u = 0; u < RU; u++) {
                const int r = r0 + u * rstep;
                x[u] = r < rows ? dense_group<BITS, ALIGNED, PREP, PM1>(codes + (long long)r * row_bytes, k0, K) : 0ull;
            }
#pragma unroll
            for (int u = 0; u < RU; u++) {
                const int r = r0 + u * rstep;
                if (r >= rows) break;
                uint32_t pw[2];
                if (BITS == 1) {
                    pw[0] = (uint32_t)x[u];
                    pw[1] = 0u;
                } else {
                    pw[0] = compress_even_bits(x[u]);
                    pw[1] = compress_even_bits(x[u] >> 1);
                }
                uint32_t* out = dst + (long long)r * BITS * Kw;
#pragma unroll
                for (int t = 0; t < BITS; t++) out[(long long)t * Kw + w] = pw[t];
                if (PREP) {
                    const int nv = K - k0;
                    const uint32_t vm = nv >= 32 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
                    uint32_t o[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const uint32_t e0 = (pw[0] >> j) & 0x11111111u, e1 = (pw[1] >> j) & 0x11111111u;
                        uint32_t v;
                        if (PM1) v = 0x22222222u | ((e0 ^ 0x11111111u) << 3);  // +1 -> 0x2, -1 -> 0xA
                        else v = (e1 << 2) | ((e0 & ~e1) << 1) | (e0 & e1);    // 0..3 -> 0x0, 0x2, 0x4, 0x5
                        o[j] = v & (((vm >> j) & 0x11111111u) * 0xFu);
                    }
                    *reinterpret_cast<uint4*>(prep + ((long long)r * Kw + w) * 16) =
                        make_uint4(o[0], o[1], o[2], o[3]);
                }
            }
        }
    }
}

template <int BITS, bool PREP, bool PM1>
static void dense_launch(bool aligned, dim3 grid, dim3 threads, cudaStream_t s, const uint8_t* codes, int rows,
                         int K, int row_bytes, int Kw, uint32_t* dst, uint8_t* prep) {
    if (aligned)
        pack_dense_kernel<BITS, true, PREP, PM1><<<grid, threads, 0, s>>>(codes, rows, K, row_bytes, Kw, dst, prep);
    else
        pack_dense_kernel<BITS, false, PREP, PM1><<<grid, threads, 0, s>>>(codes, rows, K, row_bytes, Kw, dst, prep);
}

// dense bits-per-element codes (bits 1 or 2) -> planes (+ e2m1 rows when prep != nullptr)
cudaError_t launch_pack_dense(const uint8_t* codes, int rows, int K, int bits, uint32_t* dst, int sms,
                              cudaStream_t s, uint8_t* prep, bool pm1) {
    const int Kw = (K + 127) / 128 * 4;
    if ((long long)rows * Kw == 0) return cudaSuccess;
    const int row_bytes = (K * bits + 7) / 8;
    const bool aligned = (row_bytes % (bits * 4) == 0) && ((reinterpret_cast<uintptr_t>(codes) & 7) == 0);
    dim3 threads(Kw >= 256 ? 256 : (Kw + 31) / 32 * 32, 1);
    threads.y = 256 / threads.x;
    dim3 grid((Kw + threads.x - 1) / threads.x, 1);
    const long long ry = ((long long)sms * 8 + grid.x - 1) / grid.x, need = ((long long)rows + threads.y - 1) / threads.y;
    grid.y = (unsigned)(ry < need ? ry : need);
    if (grid.y > 65535) grid.y = 65535;
    if (bits == 1) {
        if (!prep) dense_launch<1, false, false>(aligned, grid, threads, s, codes, rows, K, row_bytes, Kw, dst, prep);
        else if (pm1) dense_launch<1, true, true>(aligned, grid, threads, s, codes, rows, K, row_bytes, Kw, dst, prep);
        else dense_launch<1, true, false>(aligned, grid, threads, s, codes, rows, K, row_bytes, Kw, dst, prep);
    } else {
        if (!prep) dense_launch<2, false, false>(aligned, grid, threads, s, codes, rows, K, row_bytes, Kw, dst, prep);
        else dense_launch<2, true, false>(aligned, grid, threads, s, codes, rows, K, row_bytes, Kw, dst, prep);
    }
    count_launch();
    return cudaGetLastError();
}

template <bool PREP, bool PM1>
static void pack_launch(bool vec, dim3 grid, dim3 threads, cudaStream_t s, const uint8_t* codes, int rows, int K,
                        int bits, int Kw, uint32_t* dst, uint8_t* prep) {
    if (vec) pack_bits_kernel<true, PREP, PM1><<<grid, threads, 0, s>>>(codes, rows, K, bits, Kw, dst, prep);
    else pack_bits_kernel<false, PREP, PM1><<<grid, threads, 0, s>>>(codes, rows, K, bits, Kw, dst, prep);
}

// prep != nullptr: also the e2m1 operand rows (bits <= 2; pm1: +-1 codes)
cudaError_t launch_pack_bits(const uint8_t* codes, int rows, int K, int bits, uint32_t* dst,
                             int sms, cudaStream_t s, uint8_t* prep, bool pm1) {
    const int Kw = (K + 127) / 128 * 4;
    if ((long long)rows * Kw == 0) return cudaSuccess;
    const bool vec = (K % 16 == 0) && ((reinterpret_cast<uintptr_t>(codes) & 15) == 0);
    dim3 threads(Kw >= 256 ? 256 : (Kw + 31) / 32 * 32, 1);
    threads.y = 256 / threads.x;
    dim3 grid((Kw + threads.x - 1) / threads.x, 1);
    const long long ry = ((long long)sms * 8 + grid.x - 1) / grid.x, need = ((long long)rows + threads.y - 1) / threads.y;
    grid.y = (unsigned)(ry < need ? ry : need);
    if (grid.y > 65535) grid.y = 65535;
    if (!prep) pack_launch<false, false>(vec, grid, threads, s, codes, rows, K, bits, Kw, dst, prep);
    else if (pm1) pack_launch<true, true>(vec, grid, threads, s, codes, rows, K, bits, Kw, dst, prep);
    else pack_launch<true, false>(vec, grid, threads, s, codes, rows, K, bits, Kw, dst, prep);
    count_launch();
    return cudaGetLastError();
}
}  // namespace apnn

namespace apnn {
cudaError_t launch_im2col_pack(const uint8_t* X, int B, int H, int W, int C, int R, int S, int stride, int pad,
                               int Ho, int Wo, int bits, uint32_t* dst, int sms, cudaStream_t s, int qz, int qs) {
    const int Kw = (R * S * C + 127) / 128 * 4;
    const long long total = (long long)B * Ho * Wo;
    if (total == 0) return cudaSuccess;
    const size_t smem = (((size_t)R * (W + 2 * pad) * C + 1 + 15) & ~(size_t)15) + (size_t)Kw * 32 * 4 +
                        (size_t)Wo * bits * Kw * 4;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(im2col_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    const long long ctas = (long long)B * Ho;
    const int grid = (int)(ctas < (long long)sms * 4 ? ctas : (long long)sms * 4);
    im2col_pack_kernel<<<grid, 256, smem, s>>>(X, B, H, W, C, R, S, stride, pad, Ho, Wo, bits, Kw, dst, qz, qs);
    count_launch();
    return cudaGetLastError();
}
}  // namespace apnn

namespace apnn {
cudaError_t launch_flatten_packed(const uint32_t* src, int B, int P, int bits, int Cw, uint32_t* dst, int sms,
                                  cudaStream_t s) {
    const long long total = (long long)B * P * bits * Cw;
    if (total == 0) return cudaSuccess;
    flatten_packed_kernel<<<stream_grid(total, sms), 256, 0, s>>>(src, B, P, bits, Cw, dst);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// k x k / stride max pooling over PACKED codes (apnn_maxpool_packed).  The requantisation
// q = clamp(floor(v / S), 0, Q) is non-decreasing in v, so max-pooling the codes equals
// quantising the max-pooled v (reading R15): a conv with the fused
// requant + pack followed by this pass does max pooling of any window without the int32 map
// ever reaching HBM.  Bit-sliced: one thread owns one 32-channel word of one output pixel and
// keeps the running maximum of its window as `bits` plane words; max(x, y) per lane walks the
// planes from the MSB (x > y at the first differing plane where x has the 1).
template <int BITS>
__global__ void __launch_bounds__(256) maxpool_packed_kernel(const uint32_t* __restrict__ X, int B, int H, int W,
                                                             int Cw, int k, int stride, int Hp, int Wp,
                                                             uint32_t* __restrict__ Y) {
    const long long total = (long long)B * Hp * Wp * Cw;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int wd = (int)(idx % Cw);
        const long long pix = idx / Cw;
        const int px = (int)(pix % Wp);
        const long long t = pix / Wp;
        const int py = (int)(t % Hp);
        const int b = (int)(t / Hp);
        uint32_t m[BITS];
        const uint32_t* src = X + (((long long)b * H + (long long)py * stride) * W + (long long)px * stride) * BITS * Cw + wd;
#pragma unroll
        for (int pl = 0; pl < BITS; pl++) m[pl] = __ldg(src + pl * Cw);
        for (int dy = 0; dy < k; dy++)
            for (int dx = 0; dx < k; dx++) {
                if ((dy | dx) == 0) continue;
                const uint32_t* q = src + ((long long)dy * W + dx) * BITS * Cw;
                uint32_t x[BITS];
#pragma unroll
                for (int pl = 0; pl < BITS; pl++) x[pl] = __ldg(q + pl * Cw);
                uint32_t gt = 0u, eq = 0xFFFFFFFFu;  // lanes where x > m so far / still equal
#pragma unroll
                for (int pl = BITS - 1; pl >= 0; pl--) {
                    gt |= eq & x[pl] & ~m[pl];
                    eq &= ~(x[pl] ^ m[pl]);
                }
#pragma unroll
                for (int pl = 0; pl < BITS; pl++) m[pl] = (gt & x[pl]) | (~gt & m[pl]);
            }
        uint32_t* dst = Y + pix * BITS * Cw + wd;
#pragma unroll
        for (int pl = 0; pl < BITS; pl++) dst[pl * Cw] = m[pl];
    }
}

cudaError_t launch_maxpool_packed(const uint32_t* X, int B, int H, int W, int C, int bits, int k, int stride,
                                  uint32_t* Y, int sms, cudaStream_t s) {
    const int Cw = (C + 127) / 128 * 4;
    const int Hp = (H - k) / stride + 1, Wp = (W - k) / stride + 1;
    const long long total = (long long)B * Hp * Wp * Cw;
    if (total <= 0) return cudaSuccess;
    long long blocks = (total + 255) / 256;
    if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
    const int gb = (int)blocks;
    switch (bits) {
    case 1: maxpool_packed_kernel<1><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    case 2: maxpool_packed_kernel<2><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    case 3: maxpool_packed_kernel<3><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    case 4: maxpool_packed_kernel<4><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    case 5: maxpool_packed_kernel<5><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    case 6: maxpool_packed_kernel<6><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    case 7: maxpool_packed_kernel<7><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    default: maxpool_packed_kernel<8><<<gb, 256, 0, s>>>(X, B, H, W, Cw, k, stride, Hp, Wp, Y); break;
    }
    count_launch();
    return cudaGetLastError();
}
}  // namespace apnn

