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
#include "common.cuh"

namespace apnn {

// codes [rows][K] -> dst [rows][bits][Kw]
template <bool kVec>
__global__ void __launch_bounds__(256) pack_bits_kernel(const uint8_t* __restrict__ codes, int rows,
                                                        int K, int bits, int Kw,
                                                        uint32_t* __restrict__ dst) {
    const long long total = (long long)rows * Kw;
    const uint32_t keep = (bits >= 8) ? 0xFFFFFFFFu : (0x01010101u * ((1u << bits) - 1u));
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(idx / Kw);
        const int w = (int)(idx - (long long)r * Kw);
        const int k0 = w * 32;
        uint32_t u[8];
        if (k0 + 32 <= K) {
            const uint8_t* src = codes + (long long)r * K + k0;
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
                    if (k < K) x |= (uint32_t)codes[(long long)r * K + k] << (8 * b);
                }
                u[q] = x;
            }
        }
#pragma unroll
        for (int q = 0; q < 8; q++) u[q] &= keep;  // codes are masked to their low `bits` bits
        uint32_t* out = dst + (long long)r * bits * Kw + w;
        for (int t = 0; t < bits; t++) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) word |= byte_bits_to_nibble(u[q], t) << (4 * q);
            out[(long long)t * Kw] = word;
        }
    }
}

// Y [M][N] int32 -> out [M][ob][Nw], Nw = roundup(N,128)/32
__global__ void __launch_bounds__(256) quant_pack_kernel(const int32_t* __restrict__ Y, int M, int N,
                                                         int Nw, Epi e, uint32_t* __restrict__ out,
                                                         bool vec) {
    const long long total = (long long)M * Nw;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int m = (int)(idx / Nw);
        const int w = (int)(idx - (long long)m * Nw);
        const int n0 = w * 32;
        uint32_t qb[8];  // 32 codes, 4 per word (byte i of qb[q] = code of column n0+4q+i)
#pragma unroll
        for (int q = 0; q < 8; q++) qb[q] = 0;
        if (n0 < N) {
            const int32_t* src = Y + (long long)m * N + n0;
            if (vec && n0 + 32 <= N) {
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    int4 v = __ldg(reinterpret_cast<const int4*>(src) + q);
                    int n = n0 + 4 * q;
                    qb[q] = requant(e, v.x, epi_alpha(e, n), epi_beta(e, n)) |
                            (requant(e, v.y, epi_alpha(e, n + 1), epi_beta(e, n + 1)) << 8) |
                            (requant(e, v.z, epi_alpha(e, n + 2), epi_beta(e, n + 2)) << 16) |
                            (requant(e, v.w, epi_alpha(e, n + 3), epi_beta(e, n + 3)) << 24);
                }
            } else {
                for (int i = 0; i < 32; i++) {
                    int n = n0 + i;
                    if (n < N) qb[i >> 2] |= requant(e, __ldg(src + i), epi_alpha(e, n), epi_beta(e, n))
                                             << (8 * (i & 3));
                }
            }
        }
        uint32_t* o = out + (long long)m * e.out_bits * Nw + w;
        for (int t = 0; t < e.out_bits; t++) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) word |= byte_bits_to_nibble(qb[q], t) << (4 * q);
            o[(long long)t * Nw] = word;
        }
    }
}

// Y [B][H][W][N] int32 (NHWC conv output) -> out [B*Hp*Wp][ob][Nw]: k x k pooling of
// v = alpha*y + beta (max, or floor of the average), then quantisation and packing
// (reading R15).  One warp per (pooled pixel, output word):
// lane = channel (coalesced 128-byte loads, k*k independent loads per lane), and the
// plane words are formed with __ballot_sync as in the paper's output packing
// (PAPER.md:1582-1587).
__global__ void __launch_bounds__(256) pool_quant_pack_kernel(const int32_t* __restrict__ Y, int B, int H, int W,
                                                              int N, int Hp, int Wp, int Nw, Epi e,
                                                              uint32_t* __restrict__ out) {
    const long long total = (long long)B * Hp * Wp * Nw;  // warps of work
    const int k = e.pool, st = e.pool_stride;
    const int lane = threadIdx.x & 31;
    const long long wstride = (long long)gridDim.x * (blockDim.x / 32);
    for (long long idx = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5); idx < total;
         idx += wstride) {
        const long long pix = idx / Nw;
        const int w = (int)(idx - pix * Nw);
        const int b = (int)(pix / ((long long)Hp * Wp));
        const int rem = (int)(pix - (long long)b * Hp * Wp);
        const int i = rem / Wp, j = rem - (rem / Wp) * Wp;
        const int n = w * 32 + lane;
        uint32_t q = 0;
        if (n < N) {
            const long long al = epi_alpha(e, n), be = epi_beta(e, n);
            long long best = 0, sum = 0;
            for (int r = 0; r < k; r++) {
                const int32_t* row = Y + (((long long)b * H + i * st + r) * W + j * st) * N + n;
                for (int s2 = 0; s2 < k; s2++) {
                    const long long v = al * __ldg(row + (long long)s2 * N) + be;
                    best = (r == 0 && s2 == 0) ? v : (v > best ? v : best);
                    sum += v;
                }
            }
            long long P = best;
            if (e.pool_avg) {
                const long long kk = (long long)k * k;
                P = sum / kk;
                if (sum % kk != 0 && sum < 0) P -= 1;  // floor toward -inf
            }
            q = quantise_v(e, P);
        }
        uint32_t* o = out + pix * e.out_bits * Nw + w;
        for (int t = 0; t < e.out_bits; t++) {
            const uint32_t word = __ballot_sync(0xFFFFFFFFu, (q >> t) & 1u);
            if (lane == t) o[(long long)t * Nw] = word;
        }
    }
}

// im2col + bit decomposition + packing of NHWC uint8 codes: one thread per (row, 32-element
// word); element k = (r*S + s)*C + c of row (b, ho, wo); out-of-frame taps are code 0.
__global__ void __launch_bounds__(256) im2col_pack_kernel(const uint8_t* __restrict__ X, int B, int H, int W,
                                                          int C, int R, int S, int stride, int pad, int Ho, int Wo,
                                                          int bits, int Kw, uint32_t* __restrict__ dst) {
    const long long rows = (long long)B * Ho * Wo;
    const long long total = rows * Kw;
    const int K = R * S * C;
    const uint32_t keep = (1u << bits) - 1u;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long m = idx / Kw;
        const int w = (int)(idx - m * Kw);
        const int b = (int)(m / ((long long)Ho * Wo));
        const int rem = (int)(m - (long long)b * Ho * Wo);
        const int ho = rem / Wo, wo = rem - (rem / Wo) * Wo;
        uint32_t planes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int k = w * 32;
        int tap = k / C, c = k - tap * C;
        for (int i = 0; i < 32 && k < K; i++, k++) {
            const int r = tap / S, s2 = tap - (tap / S) * S;
            const int hi = ho * stride + r - pad, wi = wo * stride + s2 - pad;
            uint32_t code = 0;
            if (hi >= 0 && hi < H && wi >= 0 && wi < W)
                code = __ldg(X + (((long long)b * H + hi) * W + wi) * C + c) & keep;
#pragma unroll
            for (int t = 0; t < 8; t++) planes[t] |= ((code >> t) & 1u) << i;
            if (++c == C) { c = 0; tap++; }
        }
        uint32_t* o = dst + m * bits * Kw + w;
        for (int t = 0; t < bits; t++) o[(long long)t * Kw] = planes[t];
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

static int stream_grid(long long total, int sms) {
    long long blocks = (total + 255) / 256;
    long long cap = (long long)sms * 8;  // 8 resident 256-thread CTAs per SM, grid-stride beyond
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_pack_bits(const uint8_t* codes, int rows, int K, int bits, uint32_t* dst,
                             int sms, cudaStream_t s) {
    const int Kw = (K + 127) / 128 * 4;
    const long long total = (long long)rows * Kw;
    if (total == 0) return cudaSuccess;
    const bool vec = (K % 16 == 0) && ((reinterpret_cast<uintptr_t>(codes) & 15) == 0);
    if (vec)
        pack_bits_kernel<true><<<stream_grid(total, sms), 256, 0, s>>>(codes, rows, K, bits, Kw, dst);
    else
        pack_bits_kernel<false><<<stream_grid(total, sms), 256, 0, s>>>(codes, rows, K, bits, Kw, dst);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_quant_pack(const int32_t* Y, int M, int N, const Epi& e, uint32_t* out, int sms,
                              cudaStream_t s) {
    const int Nw = (N + 127) / 128 * 4;
    const long long total = (long long)M * Nw;
    if (total == 0) return cudaSuccess;
    const bool vec = (N % 4 == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
    quant_pack_kernel<<<stream_grid(total, sms), 256, 0, s>>>(Y, M, N, Nw, e, out, vec);
    count_launch();
    return cudaGetLastError();
}

}  // namespace apnn

namespace apnn {
cudaError_t launch_pool_quant_pack(const int32_t* Y, int B, int H, int W, int N, const Epi& e, uint32_t* out,
                                  int sms, cudaStream_t s) {
    const int Hp = (H - e.pool) / e.pool_stride + 1, Wp = (W - e.pool) / e.pool_stride + 1;
    const int Nw = (N + 127) / 128 * 4;
    const long long total = (long long)B * Hp * Wp * Nw;
    if (total == 0) return cudaSuccess;
    pool_quant_pack_kernel<<<stream_grid(total * 32, sms), 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
    count_launch();
    return cudaGetLastError();
}
}  // namespace apnn

namespace apnn {
cudaError_t launch_im2col_pack(const uint8_t* X, int B, int H, int W, int C, int R, int S, int stride, int pad,
                               int Ho, int Wo, int bits, uint32_t* dst, int sms, cudaStream_t s) {
    const int Kw = (R * S * C + 127) / 128 * 4;
    const long long total = (long long)B * Ho * Wo * Kw;
    if (total == 0) return cudaSuccess;
    im2col_pack_kernel<<<stream_grid(total, sms), 256, 0, s>>>(X, B, H, W, C, R, S, stride, pad, Ho, Wo, bits, Kw,
                                                               dst);
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
}  // namespace apnn
