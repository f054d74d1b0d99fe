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
#pragma unroll
                for (int i = 0; i < 32; i++) {  // static qb[] indices: no local-memory array
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
template <int KP>  // KP > 0: compile-time window (unrolled, all loads in flight); 0: runtime e.pool
__global__ void __launch_bounds__(256) pool_quant_pack_kernel(const int32_t* __restrict__ Y, int B, int H, int W,
                                                              int N, int Hp, int Wp, int Nw, Epi e,
                                                              uint32_t* __restrict__ out) {
    const int total = B * Hp * Wp * Nw;  // warps of work (host-checked < 2^31)
    const int k = KP > 0 ? KP : e.pool, st = e.pool_stride;
    const int lane = threadIdx.x & 31;
    const int wstride = gridDim.x * (blockDim.x >> 5);
    constexpr int IT = 1;  // work items per warp iteration (4 measured slower: 973 -> 1160 us on the ResNet stem)
    for (int idx0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx0 < total; idx0 += IT * wstride) {
        long long P[IT];
        int pixv[IT], wv[IT];
#pragma unroll
        for (int u = 0; u < IT; u++) {
            const int idx = idx0 + u * wstride;
            const int pix = idx / Nw;
            const int w = idx - pix * Nw;
            pixv[u] = pix;
            wv[u] = w;
            P[u] = 0;
            const int n = w * 32 + lane;
            if (idx < total && n < N) {
                const int b = pix / (Hp * Wp);
                const int rem = pix - b * Hp * Wp;
                const int i = rem / Wp, j = rem - (rem / Wp) * Wp;
                const long long al = epi_alpha(e, n), be = epi_beta(e, n);
                const int32_t* base = Y + (((long long)b * H + i * st) * W + j * st) * N + n;
                long long best = 0, sum = 0;
#pragma unroll
                for (int rr = 0; rr < k; rr++) {
#pragma unroll
                    for (int ss = 0; ss < k; ss++) {
                        const long long v = al * __ldg(base + ((long long)rr * W + ss) * N) + be;
                        best = (rr == 0 && ss == 0) ? v : (v > best ? v : best);
                        sum += v;
                    }
                }
                P[u] = best;
                if (e.pool_avg) {
                    const long long kk = (long long)k * k;
                    long long a = sum / kk;
                    if (sum % kk != 0 && sum < 0) a -= 1;  // floor toward -inf
                    P[u] = a;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < IT; u++) {
            const int idx = idx0 + u * wstride;
            if (idx >= total) break;  // warp-uniform
            const int n = wv[u] * 32 + lane;
            const uint32_t q = n < N ? quantise_v(e, P[u]) : 0u;
            uint32_t mine = 0;
#pragma unroll
            for (int t = 0; t < 8; t++) {
                if (t < e.out_bits) {
                    const uint32_t word = __ballot_sync(0xFFFFFFFFu, (q >> t) & 1u);
                    if (lane == t) mine = word;
                }
            }
            if (lane < e.out_bits) out[((long long)pixv[u] * e.out_bits + lane) * Nw + wv[u]] = mine;
        }
    }
}

// Vectorised pooling routine (N % 4 == 0): a warp handles 128 channels (4 output words) of one
// pooled pixel, lane = 4 consecutive channels (one 16-byte load per window element: 4x fewer
// load and index instructions than one channel per lane).  The 4 codes of a lane form one
// nibble per plane; 8 lanes' nibbles are OR-combined with xor-shuffles into a plane word.
template <int KP>
__global__ void __launch_bounds__(256) pool_quant_pack_v4_kernel(const int32_t* __restrict__ Y, int B, int H,
                                                                 int W, int N, int Hp, int Wp, int Nw, Epi e,
                                                                 uint32_t* __restrict__ out) {
    const int Ng = (Nw + 3) / 4;                  // 128-channel groups per pixel
    const int total = B * Hp * Wp * Ng;           // warp items (host-checked < 2^31)
    const int k = KP > 0 ? KP : e.pool, st = e.pool_stride;
    const int lane = threadIdx.x & 31;
    const int wstride = gridDim.x * (blockDim.x >> 5);
    for (int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx < total; idx += wstride) {
        const int pix = idx / Ng;
        const int grp = idx - pix * Ng;
        const int b = pix / (Hp * Wp);
        const int rem = pix - b * Hp * Wp;
        const int i = rem / Wp, j = rem - (rem / Wp) * Wp;
        const int n = grp * 128 + lane * 4;       // first of this lane's 4 channels
        uint32_t q4 = 0;                          // 4 codes, byte c = code of channel n + c
        if (n < N) {
            const int32_t* base = Y + (((long long)b * H + i * st) * W + j * st) * N + n;
            long long best[4], sum[4];
#pragma unroll
            for (int rr = 0; rr < k; rr++) {
#pragma unroll
                for (int ss = 0; ss < k; ss++) {
                    const int4 y = __ldg(reinterpret_cast<const int4*>(base + ((long long)rr * W + ss) * N));
                    const int32_t yy[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const long long v = (long long)epi_alpha(e, n + c) * yy[c] + epi_beta(e, n + c);
                        if (rr == 0 && ss == 0) { best[c] = v; sum[c] = v; }
                        else { best[c] = v > best[c] ? v : best[c]; sum[c] += v; }
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 4; c++) {
                long long P = best[c];
                if (e.pool_avg) {
                    const long long kk = (long long)k * k;
                    P = sum[c] / kk;
                    if (sum[c] % kk != 0 && sum[c] < 0) P -= 1;  // floor toward -inf
                }
                q4 |= quantise_v(e, P) << (8 * c);
            }
        }
        const int w = grp * 4 + (lane >> 3);      // output word of this lane's channels
#pragma unroll
        for (int t = 0; t < 8; t++) {
            if (t < e.out_bits) {
                uint32_t nib = byte_bits_to_nibble(q4, t) << (4 * (lane & 7));
                nib |= __shfl_xor_sync(0xFFFFFFFFu, nib, 1);
                nib |= __shfl_xor_sync(0xFFFFFFFFu, nib, 2);
                nib |= __shfl_xor_sync(0xFFFFFFFFu, nib, 4);
                if ((lane & 7) == 0 && w < Nw) out[((long long)pix * e.out_bits + t) * Nw + w] = nib;
            }
        }
    }
}

// im2col + bit decomposition + packing of NHWC uint8 codes.  One CTA per output image
// row (b, ho): the R input rows it needs are staged in shared memory with the zero
// padding materialised (R x (W + 2 pad) x C bytes, coalesced 4-byte loads), then each
// thread packs (pixel wo, word w) tasks: 32 consecutive elements k = (r*S + s)*C + c
// walked with incremental counters (no per-element division), one shared-memory byte
// read and `bits` shift-ors each; the CTA's Wo output rows are one contiguous range,
// so the words are staged in shared memory and written out coalesced.
// qs > 0: X is the raw 8-bit image and every element is quantised while it is staged,
// q = clamp(floor((x - qz) / qs), 0, 2^bits - 1) (the first layer's quantisation of the
// 8-bit input, with the quantisation formula of PAPER.md:1283-1287);
// out-of-frame taps stay code 0 (zero padding of the conv input).  qs = 0: X holds codes.
__global__ void __launch_bounds__(256) im2col_pack_kernel(const uint8_t* __restrict__ X, int B, int H, int W,
                                                          int C, int R, int S, int stride, int pad, int Ho, int Wo,
                                                          int bits, int Kw, uint32_t* __restrict__ dst, int qz,
                                                          int qs) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int Wp = W + 2 * pad, rowb = Wp * C;       // padded input row bytes
    uint8_t* rows = sm;                              // R x rowb
    uint32_t* outw = reinterpret_cast<uint32_t*>(sm + ((R * rowb + 15) & ~15));  // Wo x bits x Kw
    const int K = R * S * C;
    const uint32_t keep = (1u << bits) - 1u;
    for (int br = blockIdx.x; br < B * Ho; br += gridDim.x) {
        const int b = br / Ho, ho = br - b * Ho;
        __syncthreads();  // previous row's smem readers are done
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
            // for a filter row r the S*C codes of the window are one contiguous smem run:
            // element k = r*S*C + j sits at byte r*rowb + wo*stride*C + j
            const int SC = S * C;
            int k = w * 32;
            int r = k / SC, j = k - r * SC;
            const uint8_t* base = rows + wo * stride * C;
            int off = r * rowb + j;
            uint32_t qb[8];  // byte i of qb[j] = code of element 4j + i (as in pack_bits_kernel)
#pragma unroll
            for (int q = 0; q < 8; q++) qb[q] = 0;
#pragma unroll
            for (int e = 0; e < 32; e++) {
                if (k + e < K) qb[e >> 2] |= (uint32_t)base[off] << (8 * (e & 3));
                off++;
                if (++j == SC) { j = 0; off += rowb - SC; }
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
        uint32_t* g = dst + (long long)br * Wo * bits * Kw;  // rows (b, ho, 0..Wo-1) are contiguous
        for (int i = threadIdx.x; i < Wo * bits * Kw; i += blockDim.x) g[i] = outw[i];
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

// Residual routine: one warp per (row, 32-column word), lane = column (coalesced int32
// loads), ballot packing.  v = alpha*y + beta + rho*z in int64 (reading R24).  Each warp
// takes kItems work items per iteration and issues all their loads before any math
// (the kernel is latency-bound otherwise).
constexpr int kItems = 4;
__global__ void __launch_bounds__(256) residual_quant_pack_kernel(const int32_t* __restrict__ Y, int M, int N,
                                                                  const void* __restrict__ Z, int z_bits,
                                                                  const int32_t* __restrict__ rho, int Nw, Epi e,
                                                                  uint32_t* __restrict__ out) {
    const int total = M * Nw;  // host-checked < 2^31: 32-bit index math
    const int lane = threadIdx.x & 31;
    const int wstride = gridDim.x * (blockDim.x >> 5);
    for (int idx0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx0 < total; idx0 += kItems * wstride) {
        int32_t y[kItems];
        long long z[kItems];
        int mm[kItems], ww[kItems];
#pragma unroll
        for (int u = 0; u < kItems; u++) {
            const int idx = idx0 + u * wstride;
            mm[u] = idx / Nw;
            ww[u] = idx - mm[u] * Nw;
            const int n = ww[u] * 32 + lane;
            y[u] = 0;
            z[u] = 0;
            if (idx < total && n < N) {
                const long long m = mm[u];
                y[u] = __ldg(Y + m * N + n);
                if (z_bits == 0) {
                    z[u] = __ldg(reinterpret_cast<const int32_t*>(Z) + m * N + n);
                } else {
                    const uint32_t* zp = reinterpret_cast<const uint32_t*>(Z) + m * z_bits * Nw + ww[u];
                    uint32_t code = 0;
#pragma unroll
                    for (int t = 0; t < 8; t++)
                        if (t < z_bits) code |= ((__ldg(zp + (long long)t * Nw) >> lane) & 1u) << t;
                    z[u] = code;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kItems; u++) {
            const int idx = idx0 + u * wstride;
            if (idx >= total) break;  // warp-uniform
            const int n = ww[u] * 32 + lane;
            uint32_t q = 0;
            if (n < N) {
                const long long r = rho ? __ldg(rho + n) : 1;
                q = quantise_v(e, (long long)epi_alpha(e, n) * y[u] + epi_beta(e, n) + r * z[u]);
            }
            uint32_t mine = 0;
#pragma unroll
            for (int t = 0; t < 8; t++) {
                if (t < e.out_bits) {
                    const uint32_t word = __ballot_sync(0xFFFFFFFFu, (q >> t) & 1u);
                    if (lane == t) mine = word;
                }
            }
            if (lane < e.out_bits) out[((long long)mm[u] * e.out_bits + lane) * Nw + ww[u]] = mine;
        }
    }
}

// Vectorised residual routine (N % 4 == 0): warp = one row's 128 channels, lane = 4
// consecutive channels (16-byte loads of Y and of an int32 shortcut; packed-code shortcut: the
// lane's 4 bits of each plane word), nibbles OR-combined over 8 lanes into plane words.
__global__ void __launch_bounds__(256) residual_quant_pack_v4_kernel(const int32_t* __restrict__ Y, int M, int N,
                                                                     const void* __restrict__ Z, int z_bits,
                                                                     const int32_t* __restrict__ rho, int Nw, Epi e,
                                                                     uint32_t* __restrict__ out) {
    const int Ng = Nw / 4;
    const int total = M * Ng;  // host-checked < 2^31
    const int lane = threadIdx.x & 31;
    const int wstride = gridDim.x * (blockDim.x >> 5);
    for (int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx < total; idx += wstride) {
        const int mi = idx / Ng;
        const int grp = idx - mi * Ng;
        const long long m = mi;
        const int n = grp * 128 + lane * 4;
        const int w = grp * 4 + (lane >> 3);
        uint32_t q4 = 0;
        if (n < N) {
            const int4 y = __ldg(reinterpret_cast<const int4*>(Y + m * N + n));
            int32_t z[4];
            if (z_bits == 0) {
                const int4 zz = __ldg(reinterpret_cast<const int4*>(reinterpret_cast<const int32_t*>(Z) + m * N + n));
                z[0] = zz.x; z[1] = zz.y; z[2] = zz.z; z[3] = zz.w;
            } else {
                const uint32_t* zp = reinterpret_cast<const uint32_t*>(Z) + m * z_bits * Nw + w;
                const int sh = (lane & 7) * 4;
                uint32_t nib[8];
#pragma unroll
                for (int t = 0; t < 8; t++) nib[t] = t < z_bits ? (__ldg(zp + (long long)t * Nw) >> sh) & 0xFu : 0u;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    uint32_t code = 0;
#pragma unroll
                    for (int t = 0; t < 8; t++) code |= ((nib[t] >> c) & 1u) << t;
                    z[c] = (int32_t)code;
                }
            }
            const int32_t yy[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const long long r = rho ? __ldg(rho + n + c) : 1;
                const long long v = (long long)epi_alpha(e, n + c) * yy[c] + epi_beta(e, n + c) + r * z[c];
                q4 |= quantise_v(e, v) << (8 * c);
            }
        }
#pragma unroll
        for (int t = 0; t < 8; t++) {
            if (t < e.out_bits) {
                uint32_t nb = byte_bits_to_nibble(q4, t) << (4 * (lane & 7));
                nb |= __shfl_xor_sync(0xFFFFFFFFu, nb, 1);
                nb |= __shfl_xor_sync(0xFFFFFFFFu, nb, 2);
                nb |= __shfl_xor_sync(0xFFFFFFFFu, nb, 4);
                if ((lane & 7) == 0) out[(m * e.out_bits + t) * Nw + w] = nb;
            }
        }
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
static bool pool_v4_enabled() {  // experiment knob APNN_POOL_V4=0: one channel per lane
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_POOL_V4");
        v = s ? atoi(s) : 1;
    }
    return v != 0;
}

cudaError_t launch_pool_quant_pack(const int32_t* Y, int B, int H, int W, int N, const Epi& e, uint32_t* out,
                                  int sms, cudaStream_t s) {
    const int Hp = (H - e.pool) / e.pool_stride + 1, Wp = (W - e.pool) / e.pool_stride + 1;
    const int Nw = (N + 127) / 128 * 4;
    const long long total = (long long)B * Hp * Wp * Nw;
    if (total == 0) return cudaSuccess;
    if ((long long)B * Hp * Wp * Nw > 2147483647LL) return cudaErrorInvalidValue;
    const int grid = stream_grid(total * 32, sms);
    if (N % 4 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 && pool_v4_enabled()) {
        const long long items = (long long)B * Hp * Wp * ((Nw + 3) / 4);
        const int g4 = stream_grid(items * 32, sms);
        if (e.pool == 2) pool_quant_pack_v4_kernel<2><<<g4, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
        else if (e.pool == 3) pool_quant_pack_v4_kernel<3><<<g4, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
        else pool_quant_pack_v4_kernel<0><<<g4, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
        count_launch();
        return cudaGetLastError();
    }
    if (e.pool == 2) pool_quant_pack_kernel<2><<<grid, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
    else if (e.pool == 3) pool_quant_pack_kernel<3><<<grid, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
    else pool_quant_pack_kernel<0><<<grid, 256, 0, s>>>(Y, B, H, W, N, Hp, Wp, Nw, e, out);
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
    const size_t smem = (((size_t)R * (W + 2 * pad) * C + 15) & ~(size_t)15) + (size_t)Wo * bits * Kw * 4;
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
}  // namespace apnn

namespace apnn {
cudaError_t launch_residual_quant_pack(const int32_t* Y, int M, int N, const void* Z, int z_bits,
                                       const int32_t* rho, const Epi& e, uint32_t* out, int sms, cudaStream_t s) {
    const int Nw = (N + 127) / 128 * 4;
    const long long total = (long long)M * Nw;
    if (total == 0) return cudaSuccess;
    if (total > 2147483647LL) return cudaErrorInvalidValue;
    if (N % 4 == 0 && ((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(Z)) & 15) == 0 &&
        pool_v4_enabled()) {
        residual_quant_pack_v4_kernel<<<stream_grid((long long)M * (Nw / 4) * 32, sms), 256, 0, s>>>(
            Y, M, N, Z, z_bits, rho, Nw, e, out);
        count_launch();
        return cudaGetLastError();
    }
    residual_quant_pack_kernel<<<stream_grid(total * 32, sms), 256, 0, s>>>(Y, M, N, Z, z_bits, rho, Nw, e, out);
    count_launch();
    return cudaGetLastError();
}
}  // namespace apnn
