"""X-mask sharding of the full decomposition over the GPUs of one box.

The reference's only parallelism is a static contiguous split of the tensor-number
range over std::threads (proj/src/decompose.cpp:103-126). Here the split is over
X-masks, which is what makes the device work independent and uniform:

* rank g of P = 2^p ranks owns the X-masks whose top p bits equal g
  (x in [g 2^(N-p), (g+1) 2^(N-p)));
* its coefficients are 2^p contiguous runs of 4^(N-p) entries of the reference-ordered
  array, one per value of the Z-mask's top p bits (``pd.device.run_offset``).

Two data paths, same result bit for bit:

``mode="nccl"`` (the north star's): G is replicated by one NCCL broadcast from rank 0 over
  NVLink, every rank runs K1 (diagonal gather) + K2 (Gray-code sums) on its X-mask block, and
  the runs are gathered into rank 0's output with grouped NCCL send/recv straight into their
  final offsets (rank 0's own kernel writes its runs in place, so it moves nothing).

``mode="peer"``: rank 0's G and output are mapped into every rank with CUDA IPC
  (``pd_ipc_export``/``pd_ipc_open``). K1 gathers the rank's diagonals straight from rank 0's G
  over NVLink (1/P of G crosses the switch instead of all of it), and K2's epilogue stores the
  coefficients straight into rank 0's output (PD_LAYOUT_GLOBAL on the peer pointer), so the
  transfer is spread over the kernel instead of following it. No collective on the data path:
  host barriers order rank 0's G before the peers read it and the peers' stores before rank 0
  reads the output.

Each coefficient is computed by exactly one rank with a fixed in-kernel order, so the
result is bit-identical for every P and both modes (the reference's determinism rule,
SPEC.md:200).

Plumbing is torch.distributed (backend "nccl" on GPUs, "gloo" in the CPU tests); the
compute and the peer mapping are injectable so the host logic can be tested on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable, List, Optional, Tuple

import torch
import torch.distributed as dist

from . import _paulidecomp as _ext

# compute(N, G, x0, x_count, run_bits, dst, layout, diag) writes the coefficients of the X-mask
# block into dst: "global" = the reference-ordered array of all 4^N (rank 0 in place, or rank
# 0's array mapped into a peer), "runs" = the block's 2^run_bits runs packed back to back
# (pd_layout, include/pd_api.h). G and dst are tensors or device pointers (ints).
ShardCompute = Callable[[int, Any, int, int, int, Any, str, Optional[torch.Tensor]], None]


def run_offset(num_qubits: int, run_bits: int, shard: int, run: int) -> int:
    """Offset (in coefficients) of run `run` of X-mask shard `shard` (pd_run_offset)."""
    return int(_ext.device.run_offset(num_qubits, run_bits, shard, run))


def scratch_tensor(num_qubits: int, x_count: int, path: str, device) -> torch.Tensor:
    """Scratch of an X-mask block (pd_scratch_bytes: its diagonals plus their non-finite
    flags) as a complex128 tensor."""
    nbytes = int(_ext.device.scratch_bytes(num_qubits, x_count, path))
    return torch.empty((nbytes + 15) // 16, dtype=torch.complex128, device=device)


def _ptr(buf) -> int:
    return buf.data_ptr() if isinstance(buf, torch.Tensor) else int(buf)


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

    def compute(N, G, x0, x_count, run_bits, dst, layout, diag):
        stream = torch.cuda.current_stream().cuda_stream
        _ext.device.shard_coeffs(N, _ptr(G), x0, x_count, run_bits, _ptr(dst), layout,
                                 diag.data_ptr(), path, stream)

    return compute


class CudaIpcMapper:
    """Peer mapping through the C ABI (pd_ipc_export / pd_ipc_open / pd_ipc_close)."""

    def export(self, buf: torch.Tensor) -> Tuple[bytes, int]:
        return tuple(_ext.device.ipc_export(buf.data_ptr()))

    def open(self, handle: Tuple[bytes, int]) -> int:
        return int(_ext.device.ipc_open(handle[0], handle[1]))

    def close(self, mapped: int) -> None:
        _ext.device.ipc_close(mapped)

    def fence(self) -> None:
        """This process's device work (and its peer stores) is complete."""
        torch.cuda.synchronize()


class ShardedDecomposer:
    """One rank's share of a full decomposition (one process per GPU).

    ``out`` (rank 0 only) is the complex128 array of all 4^N coefficients in reference
    order. In NCCL mode the other ranks keep their 2^p runs in a local buffer and send them to
    rank 0; in peer mode they write into rank 0's array directly.
    """

    def __init__(self, num_qubits: int, device: torch.device, group=None,
                 compute: Optional[ShardCompute] = None, path: str = "gray", mode: str = "nccl",
                 mapper=None, buffers: bool = True):
        if mode not in ("nccl", "peer"):
            raise ValueError("mode must be 'nccl' or 'peer'")
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = ShardPlan(num_qubits, world, rank)
        self.device = device
        self.mode = mode
        self.compute = compute or device_compute(path)
        self.mapper = mapper or (CudaIpcMapper() if mode == "peer" else None)
        p = self.plan
        # buffers=False: the caller owns the scratch (diag) and, in NCCL mode, sets .local
        self.diag = scratch_tensor(num_qubits, max(p.x_count, 32), path, device) \
            if buffers and device.type == "cuda" else None
        self.local = None
        if buffers and p.rank != 0 and mode == "nccl":
            self.local = torch.empty(p.run_len << p.run_bits, dtype=torch.complex128, device=device)
        self._peer_key = None      # identity of rank 0's (G, out) currently exported / mapped
        self._peer_msg = None      # rank 0: the published handles
        self._peer_bufs = None     # other ranks: (G, out) of rank 0, mapped

    # ---------------- NCCL mode ----------------

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
            self.compute(p.num_qubits, G, p.x0, p.x_count, p.run_bits, out, "global", self.diag)
        else:
            self.compute(p.num_qubits, G, p.x0, p.x_count, p.run_bits, self.local, "runs", self.diag)

    def gather(self, out: Optional[torch.Tensor]) -> None:
        p = self.plan
        if p.world == 1:
            return
        ops = []
        if p.rank == 0:
            for src in range(1, p.world):
                for o in p.offsets(src):
                    ops.append(dist.P2POp(dist.irecv, out[o:o + p.run_len], src, group=self.group))
        else:
            for run in self.run_views():
                ops.append(dist.P2POp(dist.isend, run, 0, group=self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    # ---------------- peer mode ----------------

    def peer_buffers(self, G: torch.Tensor, out: Optional[torch.Tensor]):
        """(G, out) of rank 0 as this rank addresses them: rank 0's own tensors, mapped peer
        pointers elsewhere. Rank 0 publishes the IPC handles (a small host message, not data);
        mappings are cached until rank 0's buffers change."""
        p = self.plan
        if p.world == 1:
            return G, out
        msg = [None]
        if p.rank == 0:
            # exported on every call (cheap): the handles identify the allocations, so a buffer
            # freed and reallocated at the same address is still noticed by the peers
            hg, ho = self.mapper.export(G), self.mapper.export(out)
            key = (G.data_ptr(), out.data_ptr(), hg, ho)
            if key != self._peer_key:
                self._peer_msg = (key, hg, ho)
                self._peer_key = key
            msg = [self._peer_msg]
        dist.broadcast_object_list(msg, src=0, group=self.group)
        if p.rank == 0:
            return G, out
        key, hg, ho = msg[0]
        if key != self._peer_key:
            self.close_peers()
            self._peer_bufs = (self.mapper.open(hg), self.mapper.open(ho))
            self._peer_key = key
        return self._peer_bufs

    def close_peers(self) -> None:
        if self._peer_bufs is not None:
            for b in self._peer_bufs:
                self.mapper.close(b)
        self._peer_bufs = None
        self._peer_key = None

    def _peer_step(self, G: torch.Tensor, out: Optional[torch.Tensor]) -> None:
        p = self.plan
        g_src, dst = self.peer_buffers(G, out)
        if p.world > 1:
            if p.rank == 0:
                self.mapper.fence()         # rank 0's G is written ...
            dist.barrier(group=self.group)  # ... before any peer's K1 reads it
        self.compute(p.num_qubits, g_src, p.x0, p.x_count, p.run_bits, dst, "global", self.diag)
        if p.world > 1:
            self.mapper.fence()             # this rank's peer stores are complete ...
            dist.barrier(group=self.group)  # ... before rank 0 reads (or rewrites) the output

    def __call__(self, G: torch.Tensor, out: Optional[torch.Tensor]) -> None:
        """G: complex128 [2^N, 2^N] on this rank's device (filled on rank 0, any contents
        elsewhere; not read off rank 0 in peer mode); out: complex128 [4^N] on rank 0, None
        elsewhere."""
        if self.mode == "peer":
            self._peer_step(G, out)
            return
        self.broadcast(G)
        self.compute_local(G, out)
        self.gather(out)
