// gemm_popc.cu -- CUDA-core variant of the AP-bit contraction (APNN_VARIANT_POPC).
//
// The paper's method computed literally on the integer ALUs: for every pair of
// 1-bit planes (s, t) a bit-serial product with the operator the encodings
// select, followed by the shift-weighted combination (PAPER.md:1398-1429,
// 1449-1476):
//   Case I   (0/1 x 0/1):   y += sum_s sum_t popc(a_t AND w_s) << (s+t)
//   Case II  (+-1 x +-1):   y  = n_valid - 2 popc(a XOR w)
//   Case III (+-1 W x 0/1 A): y = 2 sum_t popc(a_t AND w^) << t  -  sum_t popc(a_t) << t   (J.X term)
//   Case III swapped (+-1 A x 0/1 W): y = 2 sum_s popc(a^ AND w_s) << s - sum_s popc(w_s) << s
// Out-of-frame conv taps are skipped through a per-row validity mask so the
// +-1 cases see the value 0 there (input-aware padding).
//
// Tiling: 64x64 output tile per 256-thread CTA, 4x4 outputs per thread, one
// 128-element chunk of every plane of both operands staged in shared memory
// per step ("batch-based double caching" level 1; the
// plane index is just a shared-memory dimension = virtual batching,
// PAPER.md:1528-1533).  The fused epilogue requantises into shared memory and
// packs 32 columns per word.
#include <cstdlib>

#include "common.cuh"

namespace apnn {

namespace {
constexpr int BM = 64, BN = 64, NT = 256;
}

// APNN_POPC_WARP=0 (read once) keeps GEMMs on the tiled popc kernel (A/B measurements)
static bool popc_warp_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("APNN_POPC_WARP");
        v = s ? atoi(s) : 1;
    }
    return v != 0;
}

template <int ENC>
__global__ void __launch_bounds__(NT) popc_gemm_kernel(const uint32_t* __restrict__ A,
                                                       const uint32_t* __restrict__ Wt, Geom g,
                                                       Epi e, void* __restrict__ Yout) {
    __shared__ uint32_t sA[8][BM][4];
    __shared__ uint32_t sB[8][BN][4];
    __shared__ uint32_t sMask[BM];
    __shared__ int sNval[BM];
    __shared__ uint8_t sQ[BM][BN];

    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int ab = g.a_bits, wb = g.w_bits;

    // loader roles: row lr of the tile, planes pg, pg+4
    const int lr = tid % 64, pg = tid / 64;
    const RowCtx rctx = make_row(g, m0 + lr);
    const int bn = n0 + lr;

    int acc[4][4], aux[4][4], rowaux[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        rowaux[i] = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = aux[i][j] = 0;
    }

    for (int kc = 0; kc < g.nchunks; kc++) {
        // ---- stage chunk kc of all planes of both operands
        int nvalid;
        const uint32_t* ap = a_chunk(A, g, rctx, kc, &nvalid);
#pragma unroll
        for (int q = 0; q < 2; q++) {
            int t = pg + 4 * q;
            if (t < ab) {
                uint4 v = make_uint4(0, 0, 0, 0);
                if (ap) v = __ldg(reinterpret_cast<const uint4*>(ap + (long long)t * g.Cw));
                *reinterpret_cast<uint4*>(&sA[t][lr][0]) = v;
            }
            if (t < wb) {
                uint4 v = make_uint4(0, 0, 0, 0);
                if (bn < g.N) v = __ldg(reinterpret_cast<const uint4*>(b_chunk(Wt, g, bn, kc) + (long long)t * g.Cw));
                *reinterpret_cast<uint4*>(&sB[t][lr][0]) = v;
            }
        }
        if (pg == 0) {
            sMask[lr] = ap ? 0xFFFFFFFFu : 0u;
            sNval[lr] = nvalid;
        }
        __syncthreads();

        // ---- bit-plane products for the 4 words of the chunk
#pragma unroll
        for (int wi = 0; wi < 4; wi++) {
            uint32_t av[4][8], bv[4][8], msk[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                msk[i] = sMask[ty + 16 * i];
#pragma unroll
                for (int t = 0; t < 8; t++) av[i][t] = (t < ab) ? sA[t][ty + 16 * i][wi] : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; j++)
#pragma unroll
                for (int s = 0; s < 8; s++) bv[j][s] = (s < wb) ? sB[s][tx + 16 * j][wi] : 0u;

            if (ENC == APNN_ENC_01_01) {
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        int y = 0;
#pragma unroll
                        for (int t = 0; t < 8; t++) {
                            if (t >= ab) break;
                            int yt = 0;
#pragma unroll
                            for (int s = 0; s < 8; s++) {
                                if (s >= wb) break;
                                yt += __popc(av[i][t] & bv[j][s]) << s;
                            }
                            y += yt << t;
                        }
                        acc[i][j] += y;
                    }
            } else if (ENC == APNN_ENC_PM1_PM1) {
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) acc[i][j] += __popc((av[i][0] ^ bv[j][0]) & msk[i]);
            } else if (ENC == APNN_ENC_W_PM1_A_01) {
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    int rp = 0;
#pragma unroll
                    for (int t = 0; t < 8; t++)
                        if (t < ab) rp += __popc(av[i][t]) << t;  // J.X
                    rowaux[i] += rp;
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        int y = 0;
#pragma unroll
                        for (int t = 0; t < 8; t++)
                            if (t < ab) y += __popc(av[i][t] & bv[j][0]) << t;
                        acc[i][j] += y;
                    }
                }
            } else {  // APNN_ENC_W_01_A_PM1
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        int y = 0, c = 0;
#pragma unroll
                        for (int s = 0; s < 8; s++)
                            if (s < wb) {
                                y += __popc(av[i][0] & bv[j][s]) << s;
                                c += __popc(bv[j][s] & msk[i]) << s;
                            }
                        acc[i][j] += y;
                        aux[i][j] += c;
                    }
            }
        }
        if (ENC == APNN_ENC_PM1_PM1) {
#pragma unroll
            for (int i = 0; i < 4; i++) rowaux[i] += sNval[ty + 16 * i];
        }
        __syncthreads();
    }

    // ---- combine the encoding correction
    int y[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (ENC == APNN_ENC_01_01) y[i][j] = acc[i][j];
            else if (ENC == APNN_ENC_PM1_PM1) y[i][j] = rowaux[i] - 2 * acc[i][j];
            else if (ENC == APNN_ENC_W_PM1_A_01) y[i][j] = 2 * acc[i][j] - rowaux[i];
            else y[i][j] = 2 * acc[i][j] - aux[i][j];
        }

    if (e.out_bits == 0) {
        int32_t* Y = reinterpret_cast<int32_t*>(Yout);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            int m = m0 + ty + 16 * i;
            if (m >= g.M) continue;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                int n = n0 + tx + 16 * j;
                if (n < g.N) Y[(long long)m * g.N + n] = y[i][j];
            }
        }
        return;
    }
    // fused element-wise routine: requantise to smem, then pack 32 columns per word
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int n = n0 + tx + 16 * j;
            uint32_t q = 0;
            if (n < g.N) q = requant(e, y[i][j], epi_alpha(e, n), epi_beta(e, n));
            sQ[ty + 16 * i][tx + 16 * j] = (uint8_t)q;
        }
    __syncthreads();
    if (tid < 2 * BM) {
        const int r = tid / 2, ws = tid % 2;
        const int m = m0 + r;
        const int Nw = (g.N + 127) / 128 * 4;
        const int word = n0 / 32 + ws;
        if (m < g.M && word < Nw) {
            const uint32_t* qrow = reinterpret_cast<const uint32_t*>(&sQ[r][ws * 32]);
            uint32_t qb[8];
#pragma unroll
            for (int q = 0; q < 8; q++) qb[q] = qrow[q];
            uint32_t* o = reinterpret_cast<uint32_t*>(Yout) + (long long)m * e.out_bits * Nw + word;
            for (int t = 0; t < e.out_bits; t++) {
                uint32_t wv = 0;
#pragma unroll
                for (int q = 0; q < 8; q++) wv |= byte_bits_to_nibble(qb[q], t) << (4 * q);
                o[(long long)t * Nw] = wv;
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Warp-level variant for GEMMs (the north star's "warp-level popc/shuffle reductions"): a warp
// owns MR rows x 32 columns of Y; lane l takes K words l, l+32, ... of every plane (coalesced
// 128-byte loads of A and W rows), accumulates the bit-plane products of all MR x 32 outputs, and
// a butterfly reduce-scatter over the warp (31 __shfl_xor per row, no shared memory) leaves
// column n0 + l of each row in lane l.  The fused epilogue then packs each plane of the 32
// requantised columns with one __ballot_sync (the paper's packing).
// Latency-scale problems (the paper's FC layers, M <= 64) need one k-word per lane per plane.
// AB = a_bits as a compile-time constant: with a runtime plane count the unrolled plane loops
// issue all 8 (predicated-off) popc steps per column (w1a2 FC 9.1 us vs 3.6 us for w1a1)
template <int ENC, int MR, int AB>
__global__ void __launch_bounds__(128) popc_warp_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ Wt,
                                                        Geom g, Epi e, void* __restrict__ Yout) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int ntn = (g.N + 31) / 32;
    const int m0 = (wid / ntn) * MR, n0 = (wid % ntn) * 32;
    if (m0 >= g.M) return;  // whole warp
    constexpr int ab = AB;
    const int wb = g.w_bits, Kw = g.Cw;
    int acc[MR][32], aux[MR][32];
#pragma unroll
    for (int r = 0; r < MR; r++)
#pragma unroll
        for (int j = 0; j < 32; j++) acc[r][j] = aux[r][j] = 0;
    int rowpop[MR];  // Case III: sum_t 2^t popc(a_t) of the row (the J.X term)
#pragma unroll
    for (int r = 0; r < MR; r++) rowpop[r] = 0;
    for (int kw = lane; kw < Kw; kw += 32) {
        uint32_t a[MR][8];
#pragma unroll
        for (int r = 0; r < MR; r++) {
            const bool in = m0 + r < g.M;
#pragma unroll
            for (int t = 0; t < 8; t++)
                a[r][t] = (t < ab && in) ? __ldg(A + ((long long)(m0 + r) * ab + t) * Kw + kw) : 0u;
        }
        if (ENC == APNN_ENC_W_PM1_A_01) {
#pragma unroll
            for (int r = 0; r < MR; r++)
#pragma unroll
                for (int t = 0; t < 8; t++)
                    if (t < ab) rowpop[r] += __popc(a[r][t]) << t;
        }
        // one plane of the 32 columns' k-word, all 32 loads issued before any use (columns past N
        // read row N-1: valid memory, and their sums are never stored)
        const uint32_t* wcol = Wt + kw;
        for (int sp = 0; sp < ((ENC == APNN_ENC_PM1_PM1 || ENC == APNN_ENC_W_PM1_A_01) ? 1 : wb); sp++) {
            uint32_t wv[32];
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const int n = min(n0 + j, g.N - 1);
                wv[j] = __ldg(wcol + ((long long)n * wb + sp) * Kw);
            }
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const uint32_t w = wv[j];
                if (ENC == APNN_ENC_01_01) {
#pragma unroll
                    for (int r = 0; r < MR; r++) {
                        int y = 0;
#pragma unroll
                        for (int t = 0; t < ab; t++) y += __popc(a[r][t] & w) << t;
                        acc[r][j] += y << sp;
                    }
                } else if (ENC == APNN_ENC_PM1_PM1) {
#pragma unroll
                    for (int r = 0; r < MR; r++) acc[r][j] += __popc(a[r][0] ^ w);
                } else if (ENC == APNN_ENC_W_PM1_A_01) {
#pragma unroll
                    for (int r = 0; r < MR; r++) {
                        int y = 0;
#pragma unroll
                        for (int t = 0; t < ab; t++) y += __popc(a[r][t] & w) << t;
                        acc[r][j] += y;
                    }
                } else {  // APNN_ENC_W_01_A_PM1
                    const int pw = __popc(w) << sp;
#pragma unroll
                    for (int r = 0; r < MR; r++) {
                        acc[r][j] += __popc(a[r][0] & w) << sp;
                        aux[r][j] += pw;
                    }
                }
            }
        }
    }
    // encoding corrections, per lane partial sums over its k-words
#pragma unroll
    for (int r = 0; r < MR; r++)
#pragma unroll
        for (int j = 0; j < 32; j++) {
            if (ENC == APNN_ENC_PM1_PM1) acc[r][j] = -2 * acc[r][j];  // K_valid added after the reduction
            else if (ENC == APNN_ENC_W_PM1_A_01) acc[r][j] = 2 * acc[r][j] - rowpop[r];
            else if (ENC == APNN_ENC_W_01_A_PM1) acc[r][j] = 2 * acc[r][j] - aux[r][j];
        }
    // butterfly reduce-scatter: after the step with distance d a lane keeps the half of its
    // values whose index has bit d equal to its own lane bit, summed with its partner's
    const int Nw = (g.N + 127) / 128 * 4;
#pragma unroll
    for (int r = 0; r < MR; r++) {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            const bool up = (lane & d) != 0;
#pragma unroll
            for (int i = 0; i < d; i++) {
                const int send = up ? acc[r][i] : acc[r][i + d];
                const int keep = up ? acc[r][i + d] : acc[r][i];
                acc[r][i] = keep + __shfl_xor_sync(0xffffffffu, send, d);
            }
        }
        const int m = m0 + r, n = n0 + lane;
        int y = acc[r][0];
        if (ENC == APNN_ENC_PM1_PM1) y += g.K;  // K_valid - 2 popc(a XOR w) (padding bits agree)
        if (m >= g.M) continue;  // uniform per row
        if (e.out_bits == 0) {
            if (n < g.N) reinterpret_cast<int32_t*>(Yout)[(long long)m * g.N + n] = y;
        } else {
            const uint32_t q = n < g.N ? requant(e, y, epi_alpha(e, n), epi_beta(e, n)) : 0u;
            uint32_t* o = reinterpret_cast<uint32_t*>(Yout) + (long long)m * e.out_bits * Nw;
            for (int t = 0; t < e.out_bits; t++) {
                const uint32_t wv = __ballot_sync(0xffffffffu, (q >> t) & 1u);
                if (lane == 0) o[(long long)t * Nw + n0 / 32] = wv;
            }
            if (n0 + 32 >= g.N && lane < Nw - (n0 / 32 + 1)) {  // N padding words of the row
                for (int t = 0; t < e.out_bits; t++) o[(long long)t * Nw + n0 / 32 + 1 + lane] = 0u;
            }
        }
    }
}

template <int MR, int AB>
static void launch_popc_warp_ab(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                                int blocks, cudaStream_t s) {
    if (g.enc == APNN_ENC_01_01) popc_warp_kernel<APNN_ENC_01_01, MR, AB><<<blocks, 128, 0, s>>>(A, W, g, e, Y);
    else popc_warp_kernel<APNN_ENC_W_PM1_A_01, MR, AB><<<blocks, 128, 0, s>>>(A, W, g, e, Y);
}

// +-1 activations have one plane (Case II, Case III swapped)
template <int MR>
static void launch_popc_warp_mr(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                                cudaStream_t s) {
    const long long warps = (long long)((g.M + MR - 1) / MR) * ((g.N + 31) / 32);
    const int blocks = (int)((warps * 32 + 127) / 128);
    if (g.enc == APNN_ENC_PM1_PM1) {
        popc_warp_kernel<APNN_ENC_PM1_PM1, MR, 1><<<blocks, 128, 0, s>>>(A, W, g, e, Y);
        return;
    }
    if (g.enc == APNN_ENC_W_01_A_PM1) {
        popc_warp_kernel<APNN_ENC_W_01_A_PM1, MR, 1><<<blocks, 128, 0, s>>>(A, W, g, e, Y);
        return;
    }
    switch (g.a_bits) {
    case 1: launch_popc_warp_ab<MR, 1>(A, W, g, e, Y, blocks, s); break;
    case 2: launch_popc_warp_ab<MR, 2>(A, W, g, e, Y, blocks, s); break;
    case 3: launch_popc_warp_ab<MR, 3>(A, W, g, e, Y, blocks, s); break;
    case 4: launch_popc_warp_ab<MR, 4>(A, W, g, e, Y, blocks, s); break;
    case 5: launch_popc_warp_ab<MR, 5>(A, W, g, e, Y, blocks, s); break;
    case 6: launch_popc_warp_ab<MR, 6>(A, W, g, e, Y, blocks, s); break;
    case 7: launch_popc_warp_ab<MR, 7>(A, W, g, e, Y, blocks, s); break;
    default: launch_popc_warp_ab<MR, 8>(A, W, g, e, Y, blocks, s); break;
    }
}

// GEMM rows per warp: MR = 1 for M <= 32, else 2
static cudaError_t launch_popc_warp(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                                   cudaStream_t s) {
    if (g.M <= 32) launch_popc_warp_mr<1>(A, W, g, e, Y, s);
    else launch_popc_warp_mr<2>(A, W, g, e, Y, s);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_popc(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                        cudaStream_t s) {
    // measured (profiles/r02_popc_time.json): the warp kernel wins for M <= 256, the tiled kernel
    // (rows share the staged W chunk) above
    if (!g.conv && g.M <= 256 && popc_warp_enabled()) return launch_popc_warp(A, W, g, e, Y, s);
    const int ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;  // packed: cover the padding words
    dim3 grid((ncols + BN - 1) / BN, (g.M + BM - 1) / BM);
    if (grid.x == 0 || grid.y == 0) return cudaSuccess;
    switch (g.enc) {
    case APNN_ENC_01_01: popc_gemm_kernel<APNN_ENC_01_01><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    case APNN_ENC_PM1_PM1: popc_gemm_kernel<APNN_ENC_PM1_PM1><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    case APNN_ENC_W_PM1_A_01: popc_gemm_kernel<APNN_ENC_W_PM1_A_01><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    default: popc_gemm_kernel<APNN_ENC_W_01_A_PM1><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace apnn
