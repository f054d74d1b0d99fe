"""Multi-process tests of the data-parallel sharding (gloo on CPU, world 2 and 3).

The CUDA kernel is replaced by the CPU oracle (test infrastructure), so these
check the host-side logic the GPU runs use: shard boundaries (including uneven
M and ranks with no rows), gather order, and that the concatenation over ranks
equals the single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2106_12169_b200 import synth
from paper_2106_12169_b200.dist import ShardedAPMM, gather_rows, row_range, shard_rows


def test_row_range_covers_exactly():
    for M in (0, 1, 7, 64, 100, 8191):
        for G in (1, 2, 3, 4, 8):
            ranges = [row_range(M, G, r) for r in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == M
            for (s0, e0), (s1, e1) in zip(ranges, ranges[1:]):
                assert e0 == s1 and s0 <= e0
    with pytest.raises(ValueError):
        row_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, M, N, K, a, w, enc, out_bits, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, W = synth.gemm_inputs(M, N, K, a, w, tag="dist")
        alpha, beta = synth.epilogue_params(N, tag="dist")

        def kernel(A_rows):
            Y = oracle.gemm(A_rows.numpy(), W, a, w, enc)
            if out_bits:
                Y = oracle.pack(oracle.epilogue(Y, alpha, beta, 9, out_bits), out_bits).view(np.int32)
            return torch.from_numpy(np.ascontiguousarray(Y))

        op = ShardedAPMM(N, K, a, w, enc, kernel=kernel)
        full = op(torch.from_numpy(A), M)                       # shard + gather
        s, e = row_range(M, world, rank)
        local = op(torch.from_numpy(A[s:e].copy()), M, gather=False, sharded_input=True)
        g2 = gather_rows(local, M)
        q.put((rank, full.numpy(), g2.numpy(), shard_rows(torch.arange(M), world, rank).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,out_bits", [(2, 64, 0), (3, 100, 0), (2, 37, 2), (3, 2, 0)])
def test_sharded_equals_single_process(world, M, out_bits):
    N, K, a, w, enc = 48, 200, 2, 1, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, a, w, enc, out_bits, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="dist")
    want = oracle.gemm(A, W, a, w, enc)
    if out_bits:
        alpha, beta = synth.epilogue_params(N, tag="dist")
        want = oracle.pack(oracle.epilogue(want, alpha, beta, 9, out_bits), out_bits).view(np.int32)
    rows = []
    for rank, full, g2, myrows in sorted(res, key=lambda x: x[0]):
        np.testing.assert_array_equal(full, want)
        np.testing.assert_array_equal(g2, want)
        rows.extend(myrows.tolist())
    assert rows == list(range(M))  # shards are contiguous, in rank order, and cover M once


def _cuda_worker(rank, world, port, M, N, K, a, w, enc, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2106_12169_b200 as ap
        torch.cuda.set_device(0)
        A, W = synth.gemm_inputs(M, N, K, a, w, tag="dist-cuda")
        op = ShardedAPMM(N, K, a, w, enc, W_planes=ap.pack_bits(torch.from_numpy(W).cuda(), w))
        cuda_rows = op.kernel  # the library path: apnn_pack_bits + apnn_gemm_ex on cuda:0
        op.kernel = lambda A_rows: cuda_rows(A_rows.cuda()).cpu()  # gloo gathers host tensors
        full = op(torch.from_numpy(A), M)
        torch.cuda.synchronize()
        q.put((rank, full.numpy(), ap.launch_count()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("M", [300, 1000])
def test_sharded_cuda_kernel_two_ranks(M):
    # both ranks drive the real CUDA kernel (cuda:0) on their row shard; the gathered result
    # equals the oracle's single-process result bit for bit
    world, N, K, a, w, enc = 2, 520, 640, 2, 1, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_worker, args=(r, world, port, M, N, K, a, w, enc, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="dist-cuda")
    want = oracle.gemm(A, W, a, w, enc)
    for rank, full, launches in res:
        assert launches >= 2  # pack + GEMM ran in this rank's library instance
        np.testing.assert_array_equal(full, want)


def test_bench_relaunches_n_ranks():
    # `python bench.py --gpus 2` outside torchrun runs 2 ranks (here the reference arm, which
    # needs no GPU: rank 0 times the oracle and prints the one JSON line, rank 1 exits 0)
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--M", "64", "--N", "64", "--K", "256", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
