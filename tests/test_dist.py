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
