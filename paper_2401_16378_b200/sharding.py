"""X-mask sharding of the full decomposition over the GPUs of one box.

The reference's only parallelism is a static contiguous split of the tensor-number
range over std::threads (proj/src/decompose.cpp:103-126). Here the split is over
X-masks, which is what makes the device work independent and uniform:

* rank g of P = 2^p ranks owns the X-masks whose top p bits equal g
  (x in [g 2^(N-p), (g+1) 2^(N-p)));
* its coefficients are 2^p contiguous runs of 4^(N-p) entries of the reference-ordered
  array, one per value of the Z-mask's top p bits (``pd.device.run_offset``).

Data paths, same result bit for bit:

``mode="nccl"`` (the north star's NCCL replication and gather, pipelined; ``NcclPipeline``):
  rank g reads only the diagonals of its own X-masks (the tiles (t ^ g, t) of G, 1/P of it),
  so instead of replicating all of G, rank 0 gathers them (K1, row-major: one contiguous
  message per rank) one X-mask block at a time and sends each rank its rows with NCCL while it
  gathers the next block. A rank walks each block as soon as its rows are in (the whole-walk
  kernel, K2s / K2s-c) and sends each finished block's coefficients to rank 0 (one NCCL message,
  unpacked into their places by a run copy kernel) while the next block computes. Only the
  first block's transfer and the last block's gather are exposed. Gray path.

``mode="nccl-serial"``: one NCCL broadcast of G from rank 0, K1 + K2 on the rank's block,
  grouped NCCL send/recv of the runs straight into rank 0's output (also the WHT path and
  N < 12 under ``mode="nccl"``).

``mode="peer"``: rank 0's G and output are mapped into every rank with CUDA IPC
  (``pd_ipc_export``/``pd_ipc_open``). K1 gathers the rank's diagonals straight from rank 0's G
  over NVLink (1/P of G crosses the switch instead of all of it), and K2's epilogue stores the
  coefficients straight into rank 0's output (PD_LAYOUT_GLOBAL on the peer pointer), so the
  transfer is spread over the kernel instead of following it. No collective on the data path:
  host barriers order rank 0's G before the peers read it and the peers' stores before rank 0
  reads the output.

Each coefficient is computed by exactly one rank with a fixed in-kernel order, so the
result is bit-identical for every P and every mode (the reference's determinism rule,
SPEC.md:200).

Plumbing is torch.distributed (backend "nccl" on GPUs, "gloo" in the CPU tests); the
compute, the device data movement and the peer mapping are injectable so the host logic can
be tested on CPU.
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
                 mapper=None, buffers: bool = True, pipeline_ops=None,
                 pipeline_blocks: Optional[List[int]] = None):
        if mode not in ("nccl", "nccl-serial", "peer"):
            raise ValueError("mode must be 'nccl', 'nccl-serial' or 'peer'")
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = ShardPlan(num_qubits, world, rank)
        self.device = device
        self.compute = compute or device_compute(path)
        self.mapper = mapper or (CudaIpcMapper() if mode == "peer" else None)
        p = self.plan
        self._peer_key = None      # identity of rank 0's (G, out) currently exported / mapped
        self._peer_msg = None      # rank 0: the published handles
        self._peer_bufs = None     # other ranks: (G, out) of rank 0, mapped
        # mode "nccl": the pipelined schedule on the Gray path, else the serial broadcast /
        # compute / gather ("nccl-serial")
        self.pipeline = None
        if mode == "nccl" and path == "gray" and world > 1 and buffers and \
                (device.type == "cuda" or pipeline_ops is not None):
            try:
                self.pipeline = NcclPipeline(p, device, group, ops=pipeline_ops, sizes=pipeline_blocks)
            except ValueError:
                self.pipeline = None
        self.mode = "nccl" if self.pipeline is not None else ("peer" if mode == "peer" else "nccl-serial")
        # serial and peer modes: buffers=False means the caller owns the scratch (diag) and, in
        # the serial NCCL mode, sets .local
        self.diag = scratch_tensor(num_qubits, max(p.x_count, 32), path, device) \
            if buffers and device.type == "cuda" and self.pipeline is None else None
        self.local = None
        if buffers and p.rank != 0 and self.mode == "nccl-serial":
            self.local = torch.empty(p.run_len << p.run_bits, dtype=torch.complex128, device=device)

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
        if self.pipeline is not None:
            self.pipeline(G, out)
            return
        self.broadcast(G)
        self.compute_local(G, out)
        self.gather(out)


# ---------------------------------------------------------------------------------------------
# Pipelined NCCL mode


class TorchP2P:
    """Point-to-point transfers of the pipeline through torch.distributed (NCCL on GPUs: issued
    on the current stream's position, which then waits for them; gloo on CPU: blocking)."""

    def __init__(self, group=None):
        self.group = group

    def exchange(self, ops_list) -> None:
        """ops_list: [("send" | "recv", tensor, peer rank)], issued as one group"""
        if not ops_list:
            return
        ps = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer, group=self.group)
              for kind, t, peer in ops_list]
        for w in dist.batch_isend_irecv(ps):
            w.wait()


class DeviceOps:
    """The device primitives of the pipeline (C ABI, include/pd_api.h) on torch CUDA streams."""

    def __init__(self, device: torch.device):
        self.device = device
        # rank 0's diagonal gathers run at high priority: their CTAs go ahead of the walk's
        self.streams = {"prod": torch.cuda.Stream(device, priority=-1),
                        "comm": torch.cuda.Stream(device),
                        "walk": torch.cuda.Stream(device),
                        "walk2": torch.cuda.Stream(device)}

    def begin(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        for st in self.streams.values():
            st.wait_stream(cur)

    def end(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        for st in self.streams.values():
            cur.wait_stream(st)

    def on(self, name: str):
        return torch.cuda.stream(self.streams[name])

    def record(self, name: str):
        ev = torch.cuda.Event()
        ev.record(self.streams[name])
        return ev

    def wait(self, name: str, ev) -> None:
        self.streams[name].wait_event(ev)

    def _s(self, name: str) -> int:
        return self.streams[name].cuda_stream

    def gather(self, st, N, G, x0, x_count, out):
        _ext.device.diag_gather(N, _ptr(G), x0, x_count, _ptr(out), self._s(st))

    def coeffs(self, st, N, diag, x0, x_count, run_bits, out, layout):
        _ext.device.xmask_coeffs(N, _ptr(diag), x0, x_count, run_bits, _ptr(out), layout, "gray",
                                 self._s(st))

    def copy_runs(self, st, src, dst, run_len, src_off, dst_off):
        _ext.device.copy_runs(_ptr(src), _ptr(dst), run_len, _ptr(src_off), _ptr(dst_off),
                              src_off.numel(), self._s(st))

    def offsets(self, values: List[int]) -> torch.Tensor:
        return torch.tensor(values, dtype=torch.int64, device=self.device)


def xmask_blocks(B: int, sizes: Optional[List[int]] = None) -> List[Tuple[int, int]]:
    """A rank's B X-masks as aligned power-of-two blocks (offset, size), the pipeline's units.
    Default (profiles/r02_pipeline.md): blocks of 2048 when a rank has >= 4096 X-masks (K2s-c
    launches: N=14 on 2 or 4 GPUs); else small first and last blocks around larger middle ones
    (N=14 on 8 GPUs: 256, 256, 512, 512, 256, 256), so that only a small block's transfer is
    exposed at either end of the step."""
    if sizes is None:
        if B >= 4096:
            sizes = [2048] * (B // 2048)
        elif B >= 1024:
            sizes = [B // 8, B // 8, B // 4, B // 4, B // 8, B // 8]
        else:
            sizes = [B // 2, B // 2] if B >= 64 else [B]
    out, off = [], 0
    for sz in sizes:
        if sz <= 0 or sz & (sz - 1) or off % sz:
            raise ValueError("X-mask blocks must be aligned powers of two")
        out.append((off, sz))
        off += sz
    if off != B:
        raise ValueError("X-mask blocks must cover the rank's X-masks")
    return out


class NcclPipeline:
    """One rank's share of a full decomposition in the pipelined NCCL mode, X-mask blocks.

    Per step, for each block j of the rank's X-masks (streams: "prod" rank 0's gathers, "comm"
    NCCL and its copies, "walk"/"walk2" alternating):
      rank 0: K1 of block j of every rank (row-major diagonals, contiguous per rank) and one NCCL
        group sending each rank its rows; its own rows are its diagonals;
      rank g: receive block j's rows straight into its diagonals;
      every rank: the whole walk of block j (K2s / K2s-c + non-finite fixup) as soon as its rows
        are in; rank 0 stores in place, the others into their run buffer, pack the block's
        2^(p+q) runs into one message and send it; rank 0 receives every rank's block j and
        unpacks its runs into their offsets (pd_run_offset) of the output.
    Exposed per step: the first block's transfer and the last block's gather.
    """

    def __init__(self, plan: ShardPlan, device, group=None, ops=None, transport=None,
                 sizes: Optional[List[int]] = None):
        self.plan = plan
        self.transport = transport or TorchP2P(group)
        self.ops = ops or DeviceOps(device)
        N, P, p, B = plan.num_qubits, plan.world, plan.run_bits, plan.x_count
        if P < 2:
            raise ValueError("the NCCL pipeline needs >= 2 ranks")
        self.blocks = xmask_blocks(B, sizes)
        dim = 1 << N
        cdt = torch.complex128
        dev = device
        low = (1 << (2 * (N - p))) - 1
        self.meta = []  # per block: (bits, run_len L, coefficients)
        for off, sz in self.blocks:
            bits = p + (B // sz).bit_length() - 1
            self.meta.append((bits, 1 << (2 * (N - bits)), sz << N))
        max_out = max(m[2] for m in self.meta)
        if plan.rank == 0:
            self.send = torch.empty(dim * dim, dtype=cdt, device=dev)  # every rank's diagonals
            self.gstage = [torch.empty((P - 1) * max_out, dtype=cdt, device=dev) for _ in range(2)]
            self.unpack_src, self.unpack_dst = [], {}
            for j, (off, sz) in enumerate(self.blocks):
                bits, L, _ = self.meta[j]
                self.unpack_src.append(self.ops.offsets([R * L for R in range(1 << bits)]))
                for r in range(1, P):
                    shard = (r * B + off) // sz
                    self.unpack_dst[(r, j)] = self.ops.offsets(
                        [run_offset(N, bits, shard, R) for R in range(1 << bits)])
        else:
            self.diag = torch.empty(B * dim, dtype=cdt, device=dev)
            self.local = torch.empty(plan.run_len << p, dtype=cdt, device=dev)
            self.sendsub = [torch.empty(max_out, dtype=cdt, device=dev) for _ in range(2)]
            self.pack_src, self.pack_dst = [], []
            for j, (off, sz) in enumerate(self.blocks):
                bits, L, _ = self.meta[j]
                shard = (plan.rank * B + off) // sz
                self.pack_src.append(self.ops.offsets(
                    [(R >> (bits - p)) * plan.run_len + (run_offset(N, bits, shard, R) & low)
                     for R in range(1 << bits)]))
                self.pack_dst.append(self.ops.offsets([R * L for R in range(1 << bits)]))

    def __call__(self, G: torch.Tensor, out: Optional[torch.Tensor]) -> None:
        plan, ops = self.plan, self.ops
        N, P, p, B = plan.num_qubits, plan.world, plan.run_bits, plan.x_count
        dim = 1 << N
        ops.begin()
        ready = []
        # ---- diagonals in, block by block
        for off, sz in self.blocks:
            if plan.rank == 0:
                for r in range(P):
                    x = r * B + off
                    ops.gather("prod", N, G, x, sz, self.send[x * dim:(x + sz) * dim])
                ev = ops.record("prod")
                ready.append(ev)
                ops.wait("comm", ev)
                with ops.on("comm"):
                    self.transport.exchange([("send", self.send[(r * B + off) * dim:(r * B + off + sz) * dim], r)
                                             for r in range(1, P)])
            else:
                with ops.on("comm"):
                    self.transport.exchange([("recv", self.diag[off * dim:(off + sz) * dim], 0)])
                ready.append(ops.record("comm"))
        # ---- the whole walk of each block as soon as its rows are in
        done = []
        for j, (off, sz) in enumerate(self.blocks):
            st = "walk" if j % 2 == 0 else "walk2"
            ops.wait(st, ready[j])
            if plan.rank == 0:
                ops.coeffs(st, N, self.send[off * dim:], off, sz, 0, out, "global")
            else:
                ops.coeffs(st, N, self.diag[off * dim:], plan.x0 + off, sz, p, self.local, "runs")
            done.append(ops.record(st))
        # ---- finished blocks to rank 0
        for j, (off, sz) in enumerate(self.blocks):
            bits, L, n_out = self.meta[j]
            ops.wait("comm", done[j])
            if plan.rank == 0:
                slot = self.gstage[j % 2]
                with ops.on("comm"):
                    self.transport.exchange([("recv", slot[(r - 1) * n_out:r * n_out], r) for r in range(1, P)])
                for r in range(1, P):
                    ops.copy_runs("comm", slot[(r - 1) * n_out:], out, L, self.unpack_src[j],
                                  self.unpack_dst[(r, j)])
            else:
                buf = self.sendsub[j % 2][:n_out]
                ops.copy_runs("comm", self.local, buf, L, self.pack_src[j], self.pack_dst[j])
                with ops.on("comm"):
                    self.transport.exchange([("send", buf, 0)])
        ops.end()
