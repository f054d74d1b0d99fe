"""Candidate tiles of the int8 kernels with Eq. TLP / Eq. CI (shared by tests/test_tuner.py and
scripts/tune_time.py)."""


def candidates(M, N, K, packed=False):
    """Eq. TLP / Eq. CI over the kernels' tiles (pair 256 x bn, one CTA 128 x bn with split z)."""
    nkb = -(-K // 128)
    nmax = 64
    while nmax < N and nmax < 256:
        nmax *= 2
    out = []
    for bn in (64, 128, 256):
        if bn > nmax:
            continue
        if M > 128 and not (packed and bn == 64 and N > 64):
            out.append((2, 256, bn, 1, 2 * (-(-M // 256)) * (-(-N // bn))))
        for z in (1, 2, 4):
            if z <= nkb and (z == 1 or bn <= 128):
                out.append((1, 128, bn, z, (-(-M // 128)) * (-(-N // bn)) * z))
    return [(k, bm, bn, z, tlp, 2.0 * bm * bn / (bm + bn)) for (k, bm, bn, z, tlp) in out]
