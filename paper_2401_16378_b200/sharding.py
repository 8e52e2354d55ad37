"""X-mask sharding of the full decomposition over the GPUs of one box.

The reference's only parallelism is a static contiguous split of the tensor-number
range over std::threads (proj/src/decompose.cpp:103-126). Here the split is over
X-masks, which is what makes the device work independent and uniform:

* rank g of P = 2^p ranks owns the X-masks whose top p bits equal g
  (x in [g 2^(N-p), (g+1) 2^(N-p)));
* its coefficients are 2^p contiguous runs of 4^(N-p) entries of the reference-ordered
  array, one per value of the Z-mask's top p bits (``pd.device.run_offset``);
* G is replicated by one NCCL broadcast from rank 0 over NVLink, every rank runs
  K1 (diagonal gather) + K2 (Gray-code sums) on its X-mask block, and the runs are
  gathered into rank 0's output with grouped NCCL send/recv straight into their final
  offsets (rank 0's own kernel writes its runs in place, so it moves nothing).

Each coefficient is computed by exactly one rank with a fixed in-kernel order, so the
result is bit-identical for every P (the reference's determinism rule).

Plumbing is torch.distributed (backend "nccl" on GPUs, "gloo" in the CPU tests); the
compute is injectable so the collective logic can be tested on CPU with a stand-in.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from . import _paulidecomp as _ext

# compute(G, x0, x_count, run_bits, dst, layout, diag) writes the coefficients of the X-mask
# block into dst: "global" = the reference-ordered array of all 4^N (rank 0, in place),
# "runs" = the block's 2^run_bits runs packed back to back (pd_layout, include/pd_api.h)
ShardCompute = Callable[[torch.Tensor, int, int, int, torch.Tensor, str, Optional[torch.Tensor]], None]


def run_offset(num_qubits: int, run_bits: int, shard: int, run: int) -> int:
    """Offset (in coefficients) of run `run` of X-mask shard `shard` (pd_run_offset)."""
    return int(_ext.device.run_offset(num_qubits, run_bits, shard, run))


@dataclass
class ShardPlan:
    num_qubits: int
    world: int
    rank: int

    def __post_init__(self) -> None:
        w = self.world
        if w < 1 or (w & (w - 1)) or w > 8:
            raise ValueError("world size must be a power of two <= 8")
        if (1 << self.num_qubits) < w:
            raise ValueError("more ranks than X-masks")
        self.run_bits = w.bit_length() - 1
        self.x_count = 1 << (self.num_qubits - self.run_bits)
        self.x0 = self.rank * self.x_count
        self.run_len = 1 << (2 * (self.num_qubits - self.run_bits))
        self.total = 1 << (2 * self.num_qubits)

    def offsets(self, shard: Optional[int] = None) -> List[int]:
        g = self.rank if shard is None else shard
        return [run_offset(self.num_qubits, self.run_bits, g, r) for r in range(1 << self.run_bits)]


def device_compute(path: str = "gray") -> ShardCompute:
    """One shard's coefficients straight from G on the current CUDA stream:
    K1 + K2 (gray) or the fused two-pass WHT (wht), via pd_shard_coeffs_device."""

    def compute(G, x0, x_count, run_bits, dst, layout, diag):
        N = int(G.shape[0]).bit_length() - 1
        stream = torch.cuda.current_stream(G.device).cuda_stream
        _ext.device.shard_coeffs(N, G.data_ptr(), x0, x_count, run_bits, dst.data_ptr(), layout,
                                 diag.data_ptr(), path, stream)

    return compute


class ShardedDecomposer:
    """One rank's share of a full decomposition (one process per GPU).

    ``out`` (rank 0 only) is the complex128 array of all 4^N coefficients in reference
    order. Other ranks keep their 2^p runs in a local buffer and send them to rank 0.
    """

    def __init__(self, num_qubits: int, device: torch.device, group=None,
                 compute: Optional[ShardCompute] = None, path: str = "gray"):
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = ShardPlan(num_qubits, world, rank)
        self.device = device
        self.compute = compute or device_compute(path)
        p = self.plan
        self.diag = torch.empty(p.x_count << num_qubits, dtype=torch.complex128, device=device) \
            if device.type == "cuda" else None
        self.local = None
        if p.rank != 0:
            self.local = torch.empty(p.run_len << p.run_bits, dtype=torch.complex128, device=device)

    def run_views(self) -> List[torch.Tensor]:
        """This (non-zero) rank's packed runs, in Z-mask top-bit order."""
        p = self.plan
        return [self.local[r * p.run_len:(r + 1) * p.run_len] for r in range(1 << p.run_bits)]

    def broadcast(self, G: torch.Tensor) -> None:
        if self.plan.world > 1:
            dist.broadcast(G, src=0, group=self.group)

    def compute_local(self, G: torch.Tensor, out: Optional[torch.Tensor]) -> None:
        p = self.plan
        if p.rank == 0:
            self.compute(G, p.x0, p.x_count, p.run_bits, out, "global", self.diag)
        else:
            self.compute(G, p.x0, p.x_count, p.run_bits, self.local, "runs", self.diag)

    def gather(self, out: Optional[torch.Tensor]) -> None:
        p = self.plan
        if p.world == 1:
            return
        ops = []
        if p.rank == 0:
            for src in range(1, p.world):
                for r, o in enumerate(p.offsets(src)):
                    ops.append(dist.P2POp(dist.irecv, out[o:o + p.run_len], src, group=self.group))
        else:
            for run in self.run_views():
                ops.append(dist.P2POp(dist.isend, run, 0, group=self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def __call__(self, G: torch.Tensor, out: Optional[torch.Tensor]) -> None:
        """G: complex128 [2^N, 2^N] on this rank's device (filled on rank 0, any contents
        elsewhere); out: complex128 [4^N] on rank 0, None elsewhere."""
        self.broadcast(G)
        self.compute_local(G, out)
        self.gather(out)
