"""Print the %globaltimer trace of CTA 0 / 1 of the halo conv kernel (dev builds, APNN_HALO_TRACE)."""
import sys
import numpy as np

NEV, N = 10, 512
names = ["prod", "fwd", "mma_w", "mma_done", "dec_go", "dec_done", "mma_c", "epi_go", "epi_done", "mma_a"]
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(2, NEV, N).astype(np.int64)
t0 = None
for cta in range(2):
    print(f"--- CTA {cta} (us at 1.9 GHz)")
    t0 = t[cta][t[cta] > 0].min()
    for e in range(NEV):
        v = t[cta, e]
        idx = np.nonzero(v)[0]
        if len(idx) == 0:
            continue
        rel = (v[idx] - t0)
        print(f"{names[e]:9s} n={len(idx):3d} " + " ".join(f"{x/1900:.2f}" for x in rel[:24]))
