"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Each result is compared with the oracle so a sanitizer run is also a
parity run.  Usage: compute-sanitizer --tool T python scripts/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

cuda = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
u32 = lambda t: t.cpu().numpy().view(np.uint32)
checks = []


def gemm_case(M, N, K, a, w, enc, variant, ob=0, prepared=None):
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="san")
    Ap, Wp = ap.pack_bits(cuda(A), a), ap.pack_bits(cuda(W), w)
    Y = oracle.gemm(A, W, a, w, enc)
    epi = None
    if ob:
        alpha, beta = synth.epilogue_params(N, tag="san")
        epi = ap.Epilogue(ob, cuda(alpha), cuda(beta), 29)
        Y = oracle.pack(oracle.epilogue(Y, alpha, beta, 29, ob), ob)
    if prepared == "fp4":
        got = ap.gemm_prepared(Ap, ap.prepare_weights(Wp, N, K, w, enc), M, N, K, a, w, enc, epi=epi)
    elif prepared == "i8":
        got = ap.gemm_prepared_i8(Ap, ap.prepare_weights_i8(Wp, N, K, w, enc), M, N, K, a, w, enc, epi=epi)
    elif prepared == "fp4ab":  # fused pack + operand rows, both-prepared FP4 pair kernel
        _, Aq = ap.pack_bits_prepared(cuda(A), a, enc)
        got = ap.gemm_prepared_ab(Aq, ap.prepare_weights(Wp, N, K, w, enc), M, N, K, a, w, enc, epi=epi)
    elif prepared == "i8ab":
        got = ap.gemm_prepared_ab_i8(ap.prepare_activations_i8(Ap, M, K, a, enc), ap.prepare_weights_i8(Wp, N, K, w, enc),
                                     M, N, K, a, w, enc, epi=epi)
    else:
        got = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant)
    torch.cuda.synchronize()
    ok = np.array_equal(u32(got) if ob else got.cpu().numpy(), Y)
    checks.append((f"gemm {M}x{N}x{K} w{w}a{a} enc{enc} {prepared or ap.variant_name(variant)} ob{ob}", ok))


def conv_case(shape, a, w, enc, ob=0, pool=0):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, R, S, a, w, tag="san")
    Y = oracle.conv2d(X, Wt, st, pad, a, w, enc)
    cs = ap.ConvShape(B, H, Wd, C, Co, R, S, st, pad)
    Xp, Wp = ap.pack_bits(cuda(X.reshape(-1, C)), a), ap.pack_bits(cuda(Wt.reshape(-1, C)), w)
    epi = None
    if ob:
        alpha, beta = synth.epilogue_params(Co, tag="san")
        epi = ap.Epilogue(ob, cuda(alpha), cuda(beta), 29, pool=pool)
        if pool:
            Y = oracle.pack(oracle.pool_epilogue(Y, alpha, beta, 29, ob, pool).reshape(-1, Co), ob)
        else:
            Y = oracle.pack(oracle.epilogue(Y.reshape(-1, Co), alpha, beta, 29, ob), ob)
    got = ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi)
    torch.cuda.synchronize()
    ok = np.array_equal(u32(got) if ob else got.cpu().numpy(), Y)
    checks.append((f"conv {shape} w{w}a{a} ob{ob} pool{pool}", ok))


gemm_case(100, 200, 300, 2, 1, 2, ap.VARIANT_TC_I8)            # tc1 (M <= 128)
gemm_case(64, 64, 1024, 2, 1, 2, ap.VARIANT_TC_I8, ob=2)       # tc1 split-K cluster
gemm_case(300, 260, 300, 2, 1, 2, ap.VARIANT_TC_I8)            # tc2 pair kernel
gemm_case(300, 260, 300, 4, 4, 0, ap.VARIANT_TC_I8, ob=4)      # tc2 fused
gemm_case(300, 300, 520, 2, 2, 0, ap.VARIANT_TC_I8, prepared="i8")
gemm_case(300, 270, 300, 2, 1, 2, ap.VARIANT_TC_FP4)           # one-CTA fp4
gemm_case(100, 270, 300, 2, 1, 2, ap.VARIANT_TC_FP4, prepared="fp4")      # one-CTA fp4 prepared
gemm_case(600, 520, 700, 2, 1, 2, ap.VARIANT_TC_FP4, ob=2, prepared="fp4")  # fp4 pair kernel
gemm_case(600, 520, 700, 2, 2, 0, ap.VARIANT_TC_FP4, prepared="fp4")        # fp4 pair kernel int32
gemm_case(600, 520, 1100, 2, 1, 2, ap.VARIANT_TC_FP4, ob=2, prepared="fp4ab")  # both prepared, fused
gemm_case(300, 260, 700, 1, 1, 1, ap.VARIANT_TC_FP4, prepared="fp4ab")        # both prepared, int32
gemm_case(600, 300, 700, 4, 4, 0, ap.VARIANT_TC_I8, ob=4, prepared="i8ab")    # int8 both prepared
gemm_case(64, 1024, 1024, 2, 1, 2, ap.VARIANT_POPC, ob=2)                     # warp popc kernel
gemm_case(70, 90, 300, 3, 2, 0, ap.VARIANT_POPC)
gemm_case(70, 90, 300, 2, 1, 2, ap.VARIANT_B1MMA)
conv_case((2, 14, 14, 64, 64, 3, 3, 1, 1), 2, 1, 2)
conv_case((2, 16, 16, 64, 64, 3, 3, 1, 1), 2, 1, 2, ob=2, pool=2)
conv_case((1, 9, 9, 70, 40, 3, 3, 2, 1), 2, 2, 0, ob=2)
# max pooling over packed codes (AlexNet 3x3/2)
Q = synth.codes((2, 13, 13, 100), 2, "san-mp")
got = ap.maxpool_packed(ap.pack_bits(cuda(Q.reshape(-1, 100)), 2), 2, 13, 13, 100, 2, 3, 2)
torch.cuda.synchronize()
checks.append(("maxpool_packed 2x13x13x100 3x3/2", np.array_equal(u32(got), oracle.pack(oracle.maxpool_codes(Q, 3, 2).reshape(-1, 100), 2))))
bad = [n for n, ok in checks if not ok]
for n, ok in checks:
    print(("ok  " if ok else "BAD ") + n)
print(f"sanitize_run: {len(checks) - len(bad)}/{len(checks)} bit-exact")
sys.exit(1 if bad else 0)
