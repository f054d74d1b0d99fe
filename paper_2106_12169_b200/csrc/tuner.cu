// tuner.cu -- the paper's TLP/CI block-tiling heuristic (row f4), adapted to
// the B200 int8 tensor-core kernels.  Host code only.
//
// Paper (Eq. TLP, Eq. CI, "Auto-tuning"): candidates b_m, b_n in {16,32,64,128};
//   TLP = (pM x qN) / (b_m x b_n),   CI = 2 b_m b_n / (b_m + b_n);
// candidates go into a priority queue ordered by TLP; if the first (highest-TLP) candidate's TLP
// is below the threshold T it is taken, otherwise candidates keep being popped while TLP >= T and
// the one with the highest CI is taken.  T = 64 on the paper's GPUs.
//
// B200 adaptation (reading R21 in DESIGN.md):
//   * the candidates are the tiles the kernels implement: the CTA-pair kernel (tc2, 256 x bn,
//     bn in {64, 128, 256}, M > 128) and the one-CTA kernel (tc1, 128 x bn) with a split-K
//     cluster of z in {1, 2, 4} CTAs along K (z <= k-blocks; z > 1 needs bn <= 128: the
//     128 x bn int32 partials live in shared memory);
//   * TLP counts CTAs: ceil(M/b_m) ceil(N/b_n) z (x 2 for a pair).  The paper's p and q count
//     the bit-plane rows of its per-plane BMMA tiles; here the planes are recombined into the
//     operand bytes first, so a tile covers M x N values whatever the bit widths;
//   * CI is the paper's Eq. CI of the output tile (split-K does not change it);
//   * T = 64, the paper's empirical value: over the measured table of every candidate on the
//     latency-scale shapes (profiles/r02_tune_time.json, scripts/tune_time.py) it gives the
//     best picks of T in {8 .. 256} (geometric mean of best/picked time 0.92; T = 148, the SM
//     count, 0.81: configurations split beyond one wave of CTAs lose);
//   * tiles wider than the next power of two >= N are not candidates (padding columns only);
//   * ties in TLP pop the higher CI first, then the smaller z, then the pair kernel.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace apnn {

struct TileCand {
    int kernel, bm, bn, z;
    long long tlp;
    double ci;
};

static bool cand_before(const TileCand& a, const TileCand& b) {  // priority-queue order
    if (a.tlp != b.tlp) return a.tlp > b.tlp;
    if (a.ci != b.ci) return a.ci > b.ci;
    if (a.z != b.z) return a.z < b.z;
    return a.kernel > b.kernel;
}

static std::vector<TileCand> tile_candidates(int M, int N, int K, bool packed) {
    std::vector<TileCand> c;
    const int nkb = (K + 127) / 128;
    const int bns[3] = {64, 128, 256};
    int nmax = 64;  // widest useful tile: the next power of two >= N (at least 64)
    while (nmax < N && nmax < 256) nmax *= 2;
    for (int bn : bns) {
        if (bn > nmax) continue;  // a tile wider than the output only adds padding columns
        if (M > 128 && !(packed && bn == 64 && N > 64)) {  // packed pair stores are >= 4 words (128 columns) wide
            TileCand t{2, 256, bn, 1, 0, 0.0};
            t.tlp = 2LL * ((M + 255) / 256) * ((N + bn - 1) / bn);
            t.ci = 2.0 * t.bm * t.bn / (t.bm + t.bn);
            c.push_back(t);
        }
        for (int z = 1; z <= 4; z *= 2) {
            if (z > nkb || (z > 1 && bn > 128)) continue;
            TileCand t{1, 128, bn, z, 0, 0.0};
            t.tlp = (long long)((M + 127) / 128) * ((N + bn - 1) / bn) * z;
            t.ci = 2.0 * t.bm * t.bn / (t.bm + t.bn);
            c.push_back(t);
        }
    }
    std::sort(c.begin(), c.end(), cand_before);
    return c;
}

TileCfg tune_tiles(int M, int N, int K, int T, bool packed) {
    std::vector<TileCand> q = tile_candidates(M, N, K, packed);
    TileCfg r{1, 128, 64, 1, 0, 0.0};
    if (q.empty()) return r;
    TileCand best = q[0];
    if (best.tlp >= T) {
        for (size_t i = 1; i < q.size() && q[i].tlp >= T; i++)
            if (q[i].ci > best.ci) best = q[i];
    }
    r.kernel = best.kernel;
    r.bm = best.bm;
    r.bn = best.bn;
    r.z = best.z;
    r.tlp = best.tlp;
    r.ci = best.ci;
    return r;
}

bool tile_cfg_valid(const TileCfg& c, int M, int N, int K, bool packed) {
    const int nkb = (K + 127) / 128;
    if (c.bn != 64 && c.bn != 128 && c.bn != 256) return false;
    if (c.kernel == 2) return c.bm == 256 && c.z == 1 && M > 128 && !(packed && c.bn == 64 && N > 64);
    if (c.kernel == 1)
        return c.bm == 128 && (c.z == 1 || c.z == 2 || c.z == 4) && c.z <= nkb && (c.z == 1 || c.bn <= 128);
    return false;
}

}  // namespace apnn
