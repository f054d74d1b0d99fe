// gemm_b1mma.cu -- the paper's own primitive on B200 (APNN_VARIANT_B1MMA).
//
// 1-bit tensor-core products through the legacy warp-level
//   mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.{and,xor}.popc
// (the sm_80 successor of the bmma_sync 8x8x128 the paper uses, PAPER.md:1398,
// 1524) with the paper's operator selection and bit
// combination in registers:
//   Case I   y += sum_{s,t} bmma_and(a_t, w_s) << (s+t)
//   Case II  y  = K - 2 bmma_xor(a, w)
//   Case III y  = 2 sum_t bmma_and(a_t, w^) << t - sum_t bmma_and(a_t, J) << t   (J = all-ones
//            fragment "cached in Tensor Core fragment")
//   swapped  y  = 2 sum_s bmma_and(a^, w_s) << s - sum_s bmma_and(J, w_s) << s
// On sm_100a ptxas lowers these to IMMA.16832.U8 subroutines,
// so this variant exists to be measured against the tcgen05 path, as the north
// star requires.  Conv with +-1 activations is not offered here (the
// out-of-frame mask would need per-row J fragments); it returns
// APNN_ERR_UNSUPPORTED and the other variants cover it.
#include "common.cuh"

namespace apnn {

namespace {
constexpr int BM = 64, BN = 64, NT = 128;
}

__device__ __forceinline__ void mma_b1(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2],
                                       bool use_xor) {
    if (use_xor)
        asm volatile(
            "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%10,%11,%12,%13};\n"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(0), "r"(0), "r"(0),
              "r"(0));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%10,%11,%12,%13};\n"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(0), "r"(0), "r"(0),
              "r"(0));
}

template <int ENC>
__global__ void __launch_bounds__(NT) b1mma_gemm_kernel(const uint32_t* __restrict__ A,
                                                        const uint32_t* __restrict__ Wt, Geom g,
                                                        Epi e, void* __restrict__ Yout) {
    // one K step = 256 bits = 2 chunks = 8 words per plane per row
    __shared__ uint32_t sA[8][BM][8 + 1];
    __shared__ uint32_t sB[8][BN][8 + 1];
    __shared__ uint8_t sQ[BM][BN];

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int wm = warp / 2, wn = warp % 2;
    const int gid = lane / 4, tig = lane % 4;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int ab = g.a_bits, wb = g.w_bits;

    // loader role: row lr, chunk half lh (2 chunks per step)
    const int lr = tid % 64, lh = tid / 64;
    const RowCtx rctx = make_row(g, m0 + lr);
    const int bn = n0 + lr;

    int acc[2][4][4], aux[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int r = 0; r < 4; r++) acc[i][j][r] = aux[i][j][r] = 0;

    const uint32_t ones[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    const uint32_t onesb[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};

    for (int kc0 = 0; kc0 < g.nchunks; kc0 += 2) {
        const int kc = kc0 + lh;
        int nvalid;
        const uint32_t* ap = (kc < g.nchunks) ? a_chunk(A, g, rctx, kc, &nvalid) : nullptr;
        for (int t = 0; t < ab; t++) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (ap) v = __ldg(reinterpret_cast<const uint4*>(ap + (long long)t * g.Cw));
            uint32_t* d = &sA[t][lr][lh * 4];
            d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        }
        for (int s = 0; s < wb; s++) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (bn < g.N && kc < g.nchunks)
                v = __ldg(reinterpret_cast<const uint4*>(b_chunk(Wt, g, bn, kc) + (long long)s * g.Cw));
            uint32_t* d = &sB[s][lr][lh * 4];
            d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        }
        __syncthreads();

        // fragments: a0 (row gid, word tig), a1 (row gid+8, word tig), a2/a3 words 4+tig; b0/b1 likewise
        for (int t = 0; t < ab; t++) {
            uint32_t af[2][4];
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const int r = wm * 32 + i * 16 + gid;
                af[i][0] = sA[t][r][tig];
                af[i][1] = sA[t][r + 8][tig];
                af[i][2] = sA[t][r][4 + tig];
                af[i][3] = sA[t][r + 8][4 + tig];
            }
            if (ENC == APNN_ENC_W_PM1_A_01) {  // J.X row term
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    int d[4];
                    mma_b1(d, af[i], onesb, false);
#pragma unroll
                    for (int r = 0; r < 4; r++) aux[i][0][r] += d[r] << t;
                }
            }
            for (int s = 0; s < wb; s++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int c = wn * 32 + j * 8 + gid;
                    uint32_t bf[2] = {sB[s][c][tig], sB[s][c][4 + tig]};
                    if (ENC == APNN_ENC_W_01_A_PM1 && t == 0) {  // J.W column term
                        int d[4];
                        mma_b1(d, ones, bf, false);
#pragma unroll
                        for (int r = 0; r < 4; r++) aux[0][j][r] += d[r] << s;
                    }
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        int d[4];
                        mma_b1(d, af[i], bf, ENC == APNN_ENC_PM1_PM1);
#pragma unroll
                        for (int r = 0; r < 4; r++) acc[i][j][r] += d[r] << (s + t);
                    }
                }
            }
        }
        __syncthreads();
    }

    // C fragment: r0 (row gid, col 2tig), r1 (gid, 2tig+1), r2 (gid+8, 2tig), r3 (gid+8, 2tig+1)
    int yv[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int r = 0; r < 4; r++) {
                if (ENC == APNN_ENC_01_01) yv[i][j][r] = acc[i][j][r];
                else if (ENC == APNN_ENC_PM1_PM1) yv[i][j][r] = g.K - 2 * acc[i][j][r];
                else if (ENC == APNN_ENC_W_PM1_A_01) yv[i][j][r] = 2 * acc[i][j][r] - aux[i][0][r];
                else yv[i][j][r] = 2 * acc[i][j][r] - aux[0][j][r];
            }

#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int lrow = wm * 32 + i * 16 + gid + (r >= 2 ? 8 : 0);
                const int lcol = wn * 32 + j * 8 + 2 * tig + (r & 1);
                const int m = m0 + lrow, n = n0 + lcol;
                if (e.out_bits == 0) {
                    if (m < g.M && n < g.N) reinterpret_cast<int32_t*>(Yout)[(long long)m * g.N + n] = yv[i][j][r];
                } else {
                    uint32_t q = 0;
                    if (n < g.N) q = requant(e, yv[i][j][r], epi_alpha(e, n), epi_beta(e, n));
                    sQ[lrow][lcol] = (uint8_t)q;
                }
            }
    if (e.out_bits == 0) return;
    __syncthreads();
    {
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

bool b1mma_supports(const Geom& g) {
    return !(g.conv && (g.enc == APNN_ENC_PM1_PM1 || g.enc == APNN_ENC_W_01_A_PM1));
}

cudaError_t launch_b1mma(const uint32_t* A, const uint32_t* W, const Geom& g, const Epi& e, void* Y,
                         cudaStream_t s) {
    const int ncols = e.out_bits ? (g.N + 127) / 128 * 128 : g.N;
    dim3 grid((ncols + BN - 1) / BN, (g.M + BM - 1) / BM);
    if (grid.x == 0 || grid.y == 0) return cudaSuccess;
    switch (g.enc) {
    case APNN_ENC_01_01: b1mma_gemm_kernel<APNN_ENC_01_01><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    case APNN_ENC_PM1_PM1: b1mma_gemm_kernel<APNN_ENC_PM1_PM1><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    case APNN_ENC_W_PM1_A_01: b1mma_gemm_kernel<APNN_ENC_W_PM1_A_01><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    default: b1mma_gemm_kernel<APNN_ENC_W_01_A_PM1><<<grid, NT, 0, s>>>(A, W, g, e, Y); break;
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace apnn
