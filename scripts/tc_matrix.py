"""Development aid: tcgen05 path vs oracle over a matrix of shapes x bit combos; prints failures only."""
import sys, os, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
shapes = [(300, 64, 1000), (300, 64, 256), (256, 64, 128), (300, 128, 1000), (300, 32, 512), (600, 256, 384)]
combos = [(1, 1, 0), (2, 1, 2), (2, 2, 0), (3, 3, 0), (4, 4, 0), (5, 5, 0), (6, 6, 0), (8, 8, 0), (8, 1, 2), (1, 8, 3)]
nf = 0
for (M, N, K), (a, w, e) in itertools.product(shapes, combos):
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="mx")
    want = oracle.gemm(A, W, a, w, e)
    Y = ap.gemm(ap.pack_bits(torch.from_numpy(A).cuda(), a), ap.pack_bits(torch.from_numpy(W).cuda(), w), M, N, K, a, w, e,
                variant=ap.VARIANT_TC_I8).cpu().numpy()
    bad = Y != want
    if bad.any():
        nf += 1
        r, c = np.nonzero(bad)
        print(f"FAIL {M}x{N}x{K} a{a} w{w} e{e}: {bad.sum()} bad, rows {r.min()}-{r.max()} ({len(set(r.tolist()))}), cols {c.min()}-{c.max()}", flush=True)
print("failures", nf)
