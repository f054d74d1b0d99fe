#!/usr/bin/env python
"""Benchmark of the APNN-TC hot path on B200 (driver contract).

Workload (BASELINE.json configs[1], the GEMM sweep the metric is quoted on;
its largest point): M = N = K = 8192, w1a2, 0/1 activations x +-1 weights
(Case III).  One step = the whole hot path over one batch:
    apnn_pack_bits_dense(A codes, a bits each)   row a1 (bit decomposition into the packed
                                                 planes) fused with row a4 on A's side (the
                                                 e2m1 operand rows, once per step instead of
                                                 once per N tile inside the GEMM)
The activations arrive as dense a-bit codes (the compact format of low-bit data: 16.8 MB for
8192^2 w1a2); --byte-codes takes one byte per code (apnn_pack_bits_prepared, 67 MB).
    apnn_gemm_prepared_ab(A op, W op, epi)       rows a2-a5 + a7 (contraction on the fp4 pipe,
                                                 exact; requant + repack fused)
W is packed and prepared once at init (weights are static).
metric: effective TOPS = 2 M N K / step time (logical integer MACs x 2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--M 8192 --N 8192 --K 8192 --a 2 --w 1 --enc 2] [--variant auto]
                  [--scaling weak|strong] [--allgather]

N > 1 runs one rank per GPU over NCCL.  Launched as `python bench.py --gpus N` (no
WORLD_SIZE in the environment) it re-launches itself under torch.distributed.run with N
ranks; under torchrun it checks WORLD_SIZE == --gpus.  --scaling weak (default): every
rank processes its own M-row batch with W replicated (no data-path collective).
--scaling strong: the global M rows are sharded across the ranks (dist.row_range);
--allgather adds the output all-gather of the north star (NCCL all_gather_into_tensor)
to every step and reports its bus bandwidth.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--N", type=int, default=8192)
    ap.add_argument("--K", type=int, default=8192)
    ap.add_argument("--a", type=int, default=2)
    ap.add_argument("--w", type=int, default=1)
    ap.add_argument("--enc", type=int, default=2)
    ap.add_argument("--out-bits", type=int, default=None, help="fused output bits (default a)")
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--allgather", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-models", action="store_true")
    ap.add_argument("--no-prepared", action="store_true", help="FP4 kernel with per-tile W recombination")
    ap.add_argument("--no-prepared-a", action="store_true",
                    help="A planes decoded inside the GEMM (apnn_gemm_prepared) instead of once per step")
    ap.add_argument("--e2e-buffers", type=int, default=2,
                    help="buffer ring depth of the e2e leg (3 and 4 measured no faster: PCIe-bound)")
    ap.add_argument("--byte-codes", action="store_true",
                    help="activations as one byte per code (apnn_pack_bits_prepared) instead of dense a-bit codes")
    ap.add_argument("--no-fused-pack", action="store_true",
                    help="apnn_pack_bits + apnn_prepare_activations as two passes instead of apnn_pack_bits_prepared")
    ap.add_argument("--model-batch", type=int, default=256, help="global batch of AlexNet / VGG-Variant")
    ap.add_argument("--resnet-batch", type=int, default=1024, help="global batch of ResNet-18 w2a8")
    return ap.parse_args()


ENC_NAME = {0: "0/1 x 0/1 (Case I)", 1: "+-1 x +-1 (Case II)", 2: "0/1 act x +-1 w (Case III)",
            3: "+-1 act x 0/1 w"}


def load_peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return None


def int8_peak_tops(peaks, fp4=False):
    """Dense tensor-core peak of the pipe the GEMM runs on: measured bf16 burst x the guide's
    nominal ratio (int8 4.5 / bf16 2.25 = 2; fp4 9 / 2.25 = 4 for the kind::mxf4 variant)."""
    r = 4.0 if fp4 else 2.0
    name = "fp4" if fp4 else "int8"
    if peaks and peaks.get("bf16_tflops"):
        return float(peaks["bf16_tflops"]) * r, f"MEASURED_PEAKS.json bf16_tflops (burst) x {r:g} (nominal {name}/bf16)"
    return 1590.0 * r, f"fallback 1.59 PFLOP/s bf16 (B200_PROFILING.md) x {r:g}"


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, n in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.004)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=1)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU oracle
def oracle_sample(A, W, args, seconds, out_bits, alpha, beta, S):
    """Time the oracle as it stands on a bounded row sample of the same workload."""
    import numpy as np
    import oracle
    threads = oracle.max_threads()
    rows = 2
    t_used = 0.0
    done_rows = 0
    while True:
        t0 = time.perf_counter()
        Ys = oracle.gemm(A[:rows], W, args.a, args.w, args.enc, threads=threads)
        q = oracle.epilogue(Ys, alpha, beta, S, out_bits)
        oracle.pack(q, out_bits)
        dt = time.perf_counter() - t0
        t_used += dt
        done_rows = rows
        if dt >= seconds * 0.5 or rows >= A.shape[0]:
            break
        rows = min(A.shape[0], max(rows * 2, int(rows * seconds / max(dt, 1e-3))))
    ops = 2.0 * done_rows * W.shape[0] * W.shape[1]
    return {"value": ops / dt / 1e12, "unit": "TOPS", "cores": threads, "kind": "oracle",
            "sample": f"{done_rows} of {A.shape[0]} rows of A x full W (N={W.shape[0]}, K={W.shape[1]}): "
                      f"oracle_gemm + oracle_epilogue + oracle_pack, {dt:.2f} s, OpenMP {threads} threads",
            "seconds": round(dt, 3)}


def run_reference(args):
    """--impl reference: the CPU oracle, timed as it stands on the host cores (rank 0 only)."""
    import numpy as np
    from paper_2106_12169_b200 import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    out_bits = args.out_bits or args.a
    A, W = synth.gemm_inputs(args.M, args.N, args.K, args.a, args.w, tag="bench")
    alpha, beta = synth.epilogue_params(args.N, tag="bench")
    S = 1 << 10
    per_step = max(0.5, min(3.0, 150.0 / max(1, args.steps + args.warmup)))
    times = []
    last = None
    for i in range(args.warmup + args.steps):
        r = oracle_sample(A, W, args, per_step, out_bits, alpha, beta, S)
        if i >= args.warmup:
            times.append(r["value"])
            last = r
    value = statistics.mean(times)
    full_step_ms = 2.0 * args.M * args.N * args.K / (value * 1e12) * 1e3  # extrapolated: work is linear in M
    line = {"metric": "effective_tops_apmm", "value": value, "unit": "TOPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": full_step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8 codes, int64 accumulate", "data": "synthetic",
            "impl": "reference",
            "extrapolated": {"ms_per_step": True, "how": "each step times the oracle on a row sample of A; the "
                             "full-M step time is the sample time x M / rows (the work is exactly linear in M)"},
            "config": {"workload": f"apmm_w{args.w}a{args.a}_{args.M}x{args.N}x{args.K}_fused_pack",
                       "M": args.M, "N": args.N, "K": args.K, "a_bits": args.a, "w_bits": args.w,
                       "encoding": ENC_NAME[args.enc]},
            "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample")} | {"value": value, "unit": "TOPS"},
            "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- end-to-end models
def time_models(args, world, rank, dev, dist):
    """BASELINE.json configs[3]/[4]: AlexNet and VGG-Variant w1a2 (global batch 256) and
    ResNet-18 w2a8 (global batch 1024) end-to-end inference, global batch sharded over the ranks (strong scaling: each rank runs batch/world images), the
    whole forward captured in one CUDA graph; latency = max over ranks of the best of 5
    replays (CUDA events).  Row f1; the logits are checked against the oracle in
    tests/test_models.py."""
    import torch
    from paper_2106_12169_b200 import synth
    from paper_2106_12169_b200.models import APNNModel, APNNResNet18
    out = {}
    for name, w, a, gb in (("alexnet", 1, 2, args.model_batch), ("vgg_variant", 1, 2, args.model_batch),
                           ("resnet18", 2, 8, args.resnet_batch)):
        per = max(1, gb // world)
        # from the raw 8-bit image: the first layer quantises it on the GPU
        q = synth.input_quant(a)
        m = (APNNResNet18(per, w, a, device=dev, input_quant=q) if name == "resnet18"
             else APNNModel(name, per, w, a, device=dev, input_quant=q))
        x = torch.from_numpy(synth.model_image(name, per, tag=f"img-rank{rank}")).to(dev)
        m.run(x)
        m.capture()
        for _ in range(3):
            m.run()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record()
            m.run()
            e1.record()
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1))
        if dist is not None:
            t = torch.tensor([best], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = float(t.item())
        macs = m.macs_per_image() * per * world
        out[f"{name}_w{w}a{a}"] = {"global_batch": per * world, "batch_per_gpu": per, "latency_ms": best,
                               "images_per_s": per * world / (best * 1e-3),
                               "effective_tops": 2.0 * macs / (best * 1e-3) / 1e12, "scaling": "strong",
                               "input": "raw 8-bit image, quantised to a_bits codes in the first layer",
                               "timing": "CUDA graph of the whole forward, best of 5, max over ranks"}
        del m
    return out


# ------------------------------------------------------------------------ ours
def run_ours(args):
    import numpy as np
    import torch
    import paper_2106_12169_b200 as ap
    from paper_2106_12169_b200 import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # communicator check: every rank contributes rank + 1 (sum = N (N + 1) / 2)
        t = torch.tensor([rank + 1], dtype=torch.int64, device=torch.device("cuda", local))
        dist.all_reduce(t)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()),
                "comm_nranks_ok": bool(int(t.item()) == world * (world + 1) // 2)}
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    M_global = args.M if args.scaling == "strong" else world * args.M
    if args.scaling == "strong":  # the global M rows sharded across the ranks (dist.row_range)
        from paper_2106_12169_b200.dist import row_range
        r0, r1 = row_range(args.M, world, rank)
        args.M = r1 - r0
    M, N, K, a, w, enc = args.M, args.N, args.K, args.a, args.w, args.enc
    out_bits = args.out_bits or a
    variant = ap.VARIANTS[args.variant]

    # weak scaling: every rank owns its own M-row batch; strong: its rows of the global
    # batch.  W replicated.
    A_np, W_np = synth.gemm_inputs(M, N, K, a, w, tag="bench")
    if rank > 0:
        A_np = synth.codes((M, K), a, f"bench-rank{rank}")
    alpha_np, beta_np = synth.epilogue_params(N, tag="bench")
    S = 1 << 10
    A_codes = torch.from_numpy(A_np).to(dev)
    W_planes = ap.pack_bits(torch.from_numpy(W_np).to(dev), w)
    # weights are static: packed -- and, for the exact-FP4 kernel, prepared
    # (operand-side combination of W, apnn_prepare_weights) -- once at init, outside the step
    W_prep = None
    if variant in (0, ap.VARIANT_TC_FP4) and ap.select_variant(M, N, K, a, w, enc, out_bits) == ap.VARIANT_TC_FP4 \
            and not args.no_prepared:
        W_prep = ap.prepare_weights(W_planes, N, K, w, enc)
    # the activations' operand rows are decoded once per step (apnn_prepare_activations, inside
    # the timed step) instead of once per N tile inside the GEMM
    prep_a = W_prep is not None and a <= 2 and not args.no_prepared_a
    A_prep = None
    epi = ap.Epilogue(out_bits, torch.from_numpy(alpha_np).to(dev), torch.from_numpy(beta_np).to(dev), S)
    A_planes = torch.empty(ap.packed_shape(M, K, a), dtype=torch.int32, device=dev)
    Y_packed = torch.empty(ap.packed_shape(M, N, out_bits), dtype=torch.int32, device=dev)
    gathered = None
    if args.allgather and dist is not None:
        from paper_2106_12169_b200.dist import gather_rows
        gathered = True
    resolved = variant if variant else ap.select_variant(M, N, K, a, w, enc, out_bits)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    if prep_a:
        A_prep = ap.prepare_activations(A_planes, M, K, a, enc)

    fused_pack = prep_a and not args.no_fused_pack
    # the fused path takes the activations in their compact host format: a-bit codes stored densely
    # (a bits per element, LSB first; 16.8 MB for 8192^2 w1a2 instead of 67 MB of one-byte codes)
    dense = fused_pack and a <= 2 and not args.byte_codes
    A_dense = torch.from_numpy(synth.dense_codes(A_np, a)).to(dev) if dense else None

    def step(ev_g0=None, ev_g1=None):
        if dense:  # one pass from the dense codes: planes (the bit decomposition) + e2m1 operand rows
            ap.pack_bits_dense(A_dense, M, K, a, enc, out=A_planes, prep=A_prep)
        elif fused_pack:  # one pass: planes (the bit decomposition) + the e2m1 operand rows
            ap.pack_bits_prepared(A_codes, a, enc, out=A_planes, prep=A_prep)
        else:
            ap.pack_bits(A_codes, a, out=A_planes)
        if prep_a and not fused_pack:
            ap.prepare_activations(A_planes, M, K, a, enc, out=A_prep.data)
        if ev_g0 is not None:
            ev_g0.record(stream)
        if prep_a:
            ap.gemm_prepared_ab(A_prep, W_prep, M, N, K, a, w, enc, epi=epi, out=Y_packed)
        elif W_prep is not None:
            ap.gemm_prepared(A_planes, W_prep, M, N, K, a, w, enc, epi=epi, out=Y_packed)
        else:
            ap.gemm(A_planes, W_planes, M, N, K, a, w, enc, epi=epi, variant=variant, out=Y_packed)
        if ev_g1 is not None:
            ev_g1.record(stream)
        if gathered is not None:  # NCCL all-gather: every rank ends with all output rows
            gather_rows(Y_packed, M_global, None)

    # correctness spot check on sampled rows against nothing but the oracle happens in tests;
    # here only warm up
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)

    K_steps = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K_steps)]
    sampler = ClockSampler(local).start()
    launches0 = ap.launch_count()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    for i in range(K_steps):
        flush.fill_(i)  # L2 flush between timed steps (outside the per-step events)
        s0, g0, g1, s1 = ev[i]
        s0.record(stream)
        step(g0, g1)
        s1.record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    launches = ap.launch_count() - launches0
    clocks = sampler.stop()
    step_ms = [e[0].elapsed_time(e[3]) for e in ev]
    gemm_ms = [e[1].elapsed_time(e[2]) for e in ev]
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K_steps
    ops = 2.0 * M * N * K
    job_ops = 2.0 * M_global * N * K  # every rank's work in one step
    value = job_ops * K_steps / (total_ms * 1e-3) / 1e12
    gemm_avg_ms = statistics.mean(gemm_ms)

    # the all-gather alone: bus bandwidth (G-1)/G * gathered bytes / t, max over ranks
    allgather = None
    if gathered is not None:
        for _ in range(3):
            gather_rows(Y_packed, M_global, None)
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            gather_rows(Y_packed, M_global, None)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t_ag = torch.tensor([e0.elapsed_time(e1) / 10], dtype=torch.float64, device=dev)
        dist.all_reduce(t_ag, op=dist.ReduceOp.MAX)
        total_bytes = M_global * Y_packed[0].numel() * 4
        allgather = {"bytes_gathered": total_bytes, "ms": float(t_ag.item()),
                     "busbw_gbs": (world - 1) / world * total_bytes / (float(t_ag.item()) * 1e-3) / 1e9}

    # ---------------- e2e: same metric through the public API with host buffers.
    # Every step copies its codes host->device (pinned) and its packed output back; the
    # transfers run on their own streams, through a ring of buffers, so step i+1's upload and step
    # i-1's download overlap step i's kernels (a serving pipeline; the bytes per step are
    # unchanged).
    e2e = None
    if not args.no_e2e:
        A_host = torch.from_numpy(synth.dense_codes(A_np, a) if dense else A_np).pin_memory()
        NB = args.e2e_buffers  # ring depth: upload of step i+1, compute of step i, download of i-1 (+ slack)
        Y_host = [torch.empty(tuple(Y_packed.shape), dtype=torch.int32).pin_memory() for _ in range(NB)]
        A_dev = [torch.empty(tuple(A_host.shape), dtype=torch.uint8, device=dev) for _ in range(NB)]
        P_dev = [torch.empty_like(A_planes) for _ in range(NB)]
        Q_dev = [ap.prepare_activations(A_planes, M, K, a, enc) for _ in range(NB)] if prep_a else None
        Y_dev = [torch.empty_like(Y_packed) for _ in range(NB)]
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()

        def e2e_steps(n):
            packed_ev, d2h_ev = [None] * NB, [None] * NB
            for i in range(n):
                b = i % NB
                with torch.cuda.stream(s_h2d):
                    if packed_ev[b] is not None:
                        s_h2d.wait_event(packed_ev[b])        # A_dev[b] consumed by the previous pack
                    A_dev[b].copy_(A_host, non_blocking=True)
                    up = ev(); up.record(s_h2d)
                stream.wait_event(up)
                if dense:
                    ap.pack_bits_dense(A_dev[b], M, K, a, enc, out=P_dev[b], prep=Q_dev[b])
                elif fused_pack:
                    ap.pack_bits_prepared(A_dev[b], a, enc, out=P_dev[b], prep=Q_dev[b])
                else:
                    ap.pack_bits(A_dev[b], a, out=P_dev[b])
                packed_ev[b] = ev(); packed_ev[b].record(stream)
                if prep_a and not fused_pack:
                    ap.prepare_activations(P_dev[b], M, K, a, enc, out=Q_dev[b].data)
                if d2h_ev[b] is not None:
                    stream.wait_event(d2h_ev[b])              # Y_dev[b] downloaded
                if prep_a:
                    ap.gemm_prepared_ab(Q_dev[b], W_prep, M, N, K, a, w, enc, epi=epi, out=Y_dev[b])
                elif W_prep is not None:
                    ap.gemm_prepared(P_dev[b], W_prep, M, N, K, a, w, enc, epi=epi, out=Y_dev[b])
                else:
                    ap.gemm(P_dev[b], W_planes, M, N, K, a, w, enc, epi=epi, variant=variant, out=Y_dev[b])
                done = ev(); done.record(stream)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(done)
                    Y_host[b].copy_(Y_dev[b], non_blocking=True)
                    d2h_ev[b] = ev(); d2h_ev[b].record(s_d2h)
            for e_ in d2h_ev:
                if e_ is not None:
                    stream.wait_event(e_)

        e2e_steps(3)
        torch.cuda.synchronize(dev)
        n_e2e = max(5, min(K_steps, 20))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist is not None:
            dist.barrier()
        e0.record(stream)
        e2e_steps(n_e2e)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": job_ops * n_e2e / (e2e_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": int(A_host.numel()), "d2h_bytes_per_step": int(Y_host[0].numel() * 4),
               "steps": n_e2e, "pipelining": f"H2D / D2H on separate streams, {NB}-deep buffer ring"}

    models = None if args.no_models else time_models(args, world, rank, dev, dist)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    fp4 = resolved == ap.VARIANT_TC_FP4
    peak, peak_src = int8_peak_tops(peaks, fp4=fp4)
    achieved = ops / (gemm_avg_ms * 1e-3) / 1e12
    # which kernel ran (the library's dispatch: prepared W with M > 128 -> the CTA-pair kernel)
    kname = ("fp4_pp_kernel" if prep_a else ("fp4_pair_kernel" if M > 128 else "fp4_kernel") if W_prep is not None
             else ap.variant_name(resolved))
    traffic = None
    try:
        summ = json.load(open(NCU_SUMMARY))
        key = f"{M}x{N}x{K}_w{w}a{a}_enc{enc}_{kname}" + ("_prepared" if W_prep is not None and not prep_a else "")
        traffic = summ.get("traffic_bytes_per_launch", {}).get(key)
    except Exception:
        pass
    micro = None  # the tensor pipe's measured issue-rate ceiling (scripts/mma_peak.cu), for context
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))["summary"]
        micro = pk["kind_mxf4_tops"] if fp4 else pk["kind_i8_tops"]
    except Exception:
        pass
    line = {
        "metric": "effective_tops_apmm", "value": value, "unit": "TOPS", "n_gpus": world, "steps": K_steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "data": "synthetic",
        # arithmetic the contraction runs in: e2m1 operands with exact fp32 accumulation (|Y| < 2^24,
        # tests/test_fp4_exact.py) on the fp4 pipe, else u8/s8 operands with int32 accumulation
        "dtype": "e2m1 (fp32 accumulate, exact integers)" if fp4 else "u8/s8 (int32 accumulate)",
        "config": {"workload": f"apmm_w{w}a{a}_{M if args.scaling == 'weak' else M_global}x{N}x{K}_fused_pack",
                   "M": M_global, "M_per_rank": M, "N": N, "K": K, "a_bits": a,
                   "w_bits": w, "encoding": ENC_NAME[enc], "out": f"packed {out_bits}-bit (fused requant)",
                   "step": ("apnn_pack_bits_dense(dense a-bit A codes -> planes + e2m1 rows) + apnn_gemm_prepared_ab "
                            "(W prepared at init)") if dense else
                           ("apnn_pack_bits_prepared(A codes -> planes + e2m1 rows) + apnn_gemm_prepared_ab "
                            "(W prepared at init)") if fused_pack else "apnn_pack_bits(A) + " + (
                       "apnn_prepare_activations(A planes) + apnn_gemm_prepared_ab (W prepared at init)" if prep_a
                       else "apnn_gemm_prepared (W prepared at init)" if W_prep is not None else "apnn_gemm_fused"),
                   "variant": ap.variant_name(resolved) + ("_prepared_ab" if prep_a else "_prepared" if W_prep is not None
                                                           else ""),
                   "parallelism": f"dp{world} (" + ("M-row batch per GPU" if args.scaling == "weak"
                                                    else "global M sharded by rows") + ", W replicated)",
                   "a_input": (f"dense {a}-bit codes, {A_dense.numel()} bytes" if dense
                               else f"one byte per code, {A_codes.numel()} bytes"),
                   "l2": "flushed (512 MB write) between timed steps", "allgather": bool(gathered is not None)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": f"{kname} (apnn {ap.variant_name(resolved)} GEMM, fused epilogue"
                               + (", prepared A and W)" if prep_a else ", prepared W)" if W_prep is not None else ")"),
                     "kernel_ms": gemm_avg_ms, "kernel_share_of_step": gemm_avg_ms / ms_per_step,
                     "peak_source": peak_src,
                     "peak_mma_microbench": micro,
                     "frac_of_mma_microbench": (achieved / micro) if micro else None,
                     "traffic_source": "profiles/ncu_summary.json (dram read+write per launch, ncu --set full)"},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches,
    }
    if models is not None:
        line["models"] = models
    if comm is not None:
        line["comm"] = comm
    if allgather is not None:
        line["allgather"] = allgather
    if not args.no_cpu and world == 1:  # the oracle beside the bench: rank 0 at N = 1 only (contract)
        line["cpu_baseline"] = oracle_sample(A_np, W_np, args, args.cpu_seconds, out_bits, alpha_np, beta_np, S)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def relaunch_distributed(args):
    """`python bench.py --gpus N` outside torchrun: run N ranks (one per GPU) under
    torch.distributed.run on this node; its ranks print as usual (rank 0 the JSON line)."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
