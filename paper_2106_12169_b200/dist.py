"""Data-parallel sharding of the AP-bit GEMM/conv across GPUs.

The path partitions naturally by rows of the activation matrix (batch rows for
FC/GEMM, whole images for conv): every rank owns a contiguous M-row shard, the
packed weights are replicated, and no data moves during compute.  The only
collective is the optional output all-gather (NCCL all_gather_into_tensor over
NVLink; gloo in the CPU tests).  Because the packed layout is row-major
([rows][bits][Kw]), a shard of A, of Y or of the packed output is one
contiguous byte range, so gathering is a single flat collective.

Shard r of M rows (world G) is rows [r*P, min((r+1)*P, M)) with P = ceil(M/G);
the all-gather pads every shard to P rows and trims the result.
"""
from __future__ import annotations

import math
from typing import Callable, Optional

import torch
import torch.distributed as dist


def row_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """[start, end) rows of shard `rank` out of `world`."""
    if world < 1 or not (0 <= rank < world) or M < 0:
        raise ValueError("bad shard arguments")
    per = math.ceil(M / world) if M else 0
    start = min(rank * per, M)
    return start, min(start + per, M)


def shard_rows(x: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """This rank's contiguous row shard of a row-major tensor (codes, planes or outputs)."""
    s, e = row_range(x.shape[0], world, rank)
    return x[s:e]


def gather_rows(local: torch.Tensor, M: int, group=None) -> torch.Tensor:
    """All-gather row shards into the full [M, ...] tensor (rank order = row order)."""
    world = dist.get_world_size(group)
    per = math.ceil(M / world) if M else 0
    buf = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]].copy_(local)
    out = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:M]


class ShardedAPMM:
    """One rank's share of Y = A . W^T with W replicated.

    `kernel(A_rows, M_rows) -> Y_rows` computes the local rows; by default it is
    the CUDA path (apnn_pack_bits + apnn_gemm_ex through the C ABI).  Tests
    inject the CPU oracle here to exercise the sharding logic without a GPU.
    """

    def __init__(self, N: int, K: int, a_bits: int, w_bits: int, enc: int,
                 W_planes: Optional[torch.Tensor] = None, epi=None, group=None,
                 kernel: Optional[Callable] = None):
        self.N, self.K, self.a_bits, self.w_bits, self.enc = N, K, a_bits, w_bits, enc
        self.W_planes = W_planes
        self.epi = epi
        self.group = group
        self.kernel = kernel or self._cuda_kernel

    def _cuda_kernel(self, A_codes: torch.Tensor) -> torch.Tensor:
        import paper_2106_12169_b200 as ap
        A_planes = ap.pack_bits(A_codes, self.a_bits)
        return ap.gemm(A_planes, self.W_planes, A_codes.shape[0], self.N, self.K, self.a_bits, self.w_bits,
                       self.enc, epi=self.epi)

    def local(self, A_codes_full_or_shard: torch.Tensor, M: int, sharded_input: bool = False) -> torch.Tensor:
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        A_local = A_codes_full_or_shard if sharded_input else shard_rows(A_codes_full_or_shard, world, rank)
        s, e = row_range(M, world, rank)
        assert A_local.shape[0] == e - s
        return self.kernel(A_local)

    def __call__(self, A_codes: torch.Tensor, M: int, gather: bool = True, sharded_input: bool = False):
        y = self.local(A_codes, M, sharded_input)
        if gather and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            return gather_rows(y, M, self.group)
        return y
