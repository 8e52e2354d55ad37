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
  rank g reads only the diagonals of its X-masks, i.e. the tiles (t ^ g, t) of G — 1/P of it.
  Rank 0 gathers every rank's diagonals (K1) one walk chunk of columns at a time, in walk
  order, into a tiled buffer where each (rank, chunk) piece is contiguous, and sends each rank
  its piece with NCCL while it gathers the next chunk. A rank walks each chunk as it arrives
  (walk segments chained through raw partial sums, bit-identical to one launch, as in the host
  pipeline of pd_api.cu), finishes its X-masks in sub-blocks, and sends each finished
  sub-block's coefficients to rank 0 (one NCCL message, unpacked into their places by a run
  copy kernel) while the next sub-block computes. Gray path, N >= 12.

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
                 pipeline_chunk_log: Optional[int] = None, pipeline_sub_bits: Optional[int] = None):
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
        # mode "nccl": the pipelined schedule where it applies (Gray path, >= 4 walk chunks),
        # else the serial broadcast / compute / gather ("nccl-serial")
        self.pipeline = None
        if mode == "nccl" and path == "gray" and world > 1 and buffers and \
                (device.type == "cuda" or pipeline_ops is not None):
            try:
                self.pipeline = NcclPipeline(p, device, group, ops=pipeline_ops,
                                             chunk_log=pipeline_chunk_log, sub_bits=pipeline_sub_bits)
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


def gray(k: int) -> int:
    return k ^ (k >> 1)


def walk_segments(nch: int, ones: int = 4, runlen: int = 2) -> List[int]:
    """Chunk boundaries of the walk segments (decompose_host, pd_api.cu): the first half of the
    walk in `ones` single chunks, then aligned runs of `runlen`, so that the walk follows the
    arriving chunks; the second half (the expensive one: the most live chains) is one final
    segment per sub-block."""
    bnd, c, half = [0], 0, nch // 2
    while c < half:
        L = 1 if len(bnd) - 1 < ones else runlen
        while L > 1 and (c % L or c + L > half):
            L >>= 1
        c += L
        bnd.append(c)
    bnd.append(nch)
    return bnd


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

    def segment_chunks(self, N: int, chunk_log: int) -> int:
        return int(_ext.device.gray_segment_chunks(N, chunk_log))

    def gather_tiled(self, st, N, G, x0, x_count, col0, cols, xb_log, cb_log, out):
        _ext.device.diag_gather_tiled(N, _ptr(G), x0, x_count, col0, cols, xb_log, cb_log,
                                      _ptr(out), self._s(st))

    def place_cols(self, st, N, packed, x_count, col0, cols, diag):
        _ext.device.place_cols(N, _ptr(packed), x_count, col0, cols, _ptr(diag), self._s(st))

    def segment(self, st, N, diag, x0, x_count, chunk_log, c0, c1, part_in, part_out, run_bits,
                out, layout):
        _ext.device.gray_segment(N, _ptr(diag), x0, x_count, chunk_log, c0, c1,
                                 _ptr(part_in) if part_in is not None else 0,
                                 _ptr(part_out) if part_out is not None else 0, run_bits,
                                 _ptr(out) if out is not None else 0, layout, self._s(st))

    def copy_runs(self, st, src, dst, run_len, src_off, dst_off):
        _ext.device.copy_runs(_ptr(src), _ptr(dst), run_len, _ptr(src_off), _ptr(dst_off),
                              src_off.numel(), self._s(st))

    def offsets(self, values: List[int]) -> torch.Tensor:
        return torch.tensor(values, dtype=torch.int64, device=self.device)


class NcclPipeline:
    """One rank's share of a full decomposition in the pipelined NCCL mode (module docstring).

    Per step (streams: "prod" rank 0's gathers, "comm" NCCL and its copies, "walk"/"walk2"):
      rank 0, chunk k in walk order (columns gray(k) C .. + C): K1 of every rank's X-masks into
        the tiled send buffer, its own piece copied into its diagonals, the others' pieces sent
        (one NCCL group per chunk);
      rank g: receive chunk k, copy it into its diagonals' columns;
      every rank: walk segments over the first half as chunks arrive (raw partial sums), then
        the final segment per sub-block of 2^(N-p-q) X-masks: rank 0 writes its coefficients in
        place, the others into their run buffer, pack the sub-block's 2^(p+q) runs into one
        message and send it; rank 0 receives every rank's sub-block and unpacks its runs into
        their offsets (pd_run_offset) of the output.
    """

    CHUNK_LOG = 10  # walk chunks of 1024 steps (the host pipeline's; 1/16 of the walk at N=14)

    def __init__(self, plan: ShardPlan, device, group=None, ops=None, chunk_log: Optional[int] = None,
                 sub_bits: Optional[int] = None, transport=None):
        self.plan = plan
        self.transport = transport or TorchP2P(group)
        self.ops = ops or DeviceOps(device)
        N, P, p, B = plan.num_qubits, plan.world, plan.run_bits, plan.x_count
        self.chunk_log = self.CHUNK_LOG if chunk_log is None else chunk_log
        self.nch = self.ops.segment_chunks(N, self.chunk_log)
        if P < 2 or self.nch < 4:
            raise ValueError("the NCCL pipeline needs >= 2 ranks and >= 4 walk chunks")
        self.C = 1 << self.chunk_log
        self.bnd = walk_segments(self.nch)
        # sub-blocks of >= 256 X-masks (the host pipeline's final launches are 512 at N=14)
        self.q = (2 if B >= 1024 else (1 if B >= 256 else 0)) if sub_bits is None else sub_bits
        if (B >> self.q) < 1 or p + self.q > 8:
            raise ValueError("sub-block bits out of range")
        self.Q = 1 << self.q
        self.Bs = B >> self.q                           # X-masks per sub-block
        self.L = 1 << (2 * (N - p - self.q))            # coefficients per sub-block run
        self.sub_len = self.L << (p + self.q)           # coefficients per sub-block
        dim = 1 << N
        cdt = torch.complex128
        dev = device
        self.diag = torch.empty(B * dim, dtype=cdt, device=dev)
        self.part = torch.empty(B * dim, dtype=cdt, device=dev)
        nruns = 1 << (p + self.q)
        if plan.rank == 0:
            self.send = torch.empty(dim * dim, dtype=cdt, device=dev)
            self.gstage = [torch.empty((P - 1) * self.sub_len, dtype=cdt, device=dev) for _ in range(2)]
            # unpack: run R of rank r's sub-block s (packed at R L) -> pd_run_offset(N, p+q, rQ+s, R)
            self.unpack_src = self.ops.offsets([R * self.L for R in range(nruns)])
            self.unpack_dst = {(r, s): self.ops.offsets(
                [run_offset(N, p + self.q, r * self.Q + s, R) for R in range(nruns)])
                for r in range(1, P) for s in range(self.Q)}
        else:
            self.stage = [torch.empty(B * self.C, dtype=cdt, device=dev) for _ in range(2)]
            self.local = torch.empty(plan.run_len << p, dtype=cdt, device=dev)
            self.sendsub = [torch.empty(self.sub_len, dtype=cdt, device=dev) for _ in range(2)]
            # pack: run R = (r, u) of sub-block s, inside the rank's run r at the low 2(N-p)
            # digits of its global offset -> R L of the message
            low = (1 << (2 * (N - p))) - 1
            self.pack_src = {s: self.ops.offsets(
                [(R >> self.q) * plan.run_len + (run_offset(N, p + self.q, plan.rank * self.Q + s, R) & low)
                 for R in range(nruns)]) for s in range(self.Q)}
            self.pack_dst = self.ops.offsets([R * self.L for R in range(nruns)])

    # the send buffer's piece for (rank, column block b): tiled layout, rank block first
    def _piece(self, rank: int, b: int) -> torch.Tensor:
        B, C, nb = self.plan.x_count, self.C, self.nch
        o = (rank * nb + b) * B * C
        return self.send[o:o + B * C]


    def __call__(self, G: torch.Tensor, out: Optional[torch.Tensor]) -> None:
        plan, ops = self.plan, self.ops
        N, P, p, B = plan.num_qubits, plan.world, plan.run_bits, plan.x_count
        C, nch, bnd = self.C, self.nch, self.bnd
        dim = 1 << N
        xb_log = N - p
        ops.begin()
        ready = []
        # ---- diagonals in, walk order
        for k in range(nch):
            b = gray(k)
            if plan.rank == 0:
                ops.gather_tiled("prod", N, G, 0, dim, b * C, C, xb_log, self.chunk_log, self.send)
                ops.place_cols("prod", N, self._piece(0, b), B, b * C, C, self.diag)
                ev = ops.record("prod")
                ready.append(ev)
                ops.wait("comm", ev)
                with ops.on("comm"):
                    self.transport.exchange([("send", self._piece(r, b), r) for r in range(1, P)])
            else:
                st = self.stage[k % 2]
                with ops.on("comm"):
                    self.transport.exchange([("recv", st, 0)])
                ops.place_cols("comm", N, st, B, b * C, C, self.diag)
                ready.append(ops.record("comm"))
        # ---- first half of the walk, segment by segment as the chunks arrive
        for sg in range(len(bnd) - 2):
            ops.wait("walk", ready[bnd[sg + 1] - 1])
            ops.segment("walk", N, self.diag, plan.x0, B, self.chunk_log, bnd[sg], bnd[sg + 1],
                        self.part if sg else None, self.part, 0, None, "global")
        ops.wait("walk", ready[nch - 1])
        ops.wait("walk2", ops.record("walk"))
        # ---- final segments per sub-block; each finished sub-block goes to rank 0
        done = []
        for s in range(self.Q):
            st = "walk" if s % 2 == 0 else "walk2"
            xs = plan.x0 + s * self.Bs
            d0 = s * self.Bs * dim
            if plan.rank == 0:
                ops.segment(st, N, self.diag[d0:], xs, self.Bs, self.chunk_log, bnd[-2], 0,
                            self.part[d0:], None, 0, out, "global")
            else:
                ops.segment(st, N, self.diag[d0:], xs, self.Bs, self.chunk_log, bnd[-2], 0,
                            self.part[d0:], None, p, self.local, "runs")
            done.append(ops.record(st))
        for s in range(self.Q):
            ops.wait("comm", done[s])
            if plan.rank == 0:
                slot = self.gstage[s % 2]
                with ops.on("comm"):
                    self.transport.exchange([("recv", slot[(r - 1) * self.sub_len:r * self.sub_len], r)
                                             for r in range(1, P)])
                for r in range(1, P):
                    ops.copy_runs("comm", slot[(r - 1) * self.sub_len:], out, self.L, self.unpack_src,
                                  self.unpack_dst[(r, s)])
            else:
                buf = self.sendsub[s % 2]
                ops.copy_runs("comm", self.local, buf, self.L, self.pack_src[s], self.pack_dst)
                with ops.on("comm"):
                    self.transport.exchange([("send", buf, 0)])
        ops.end()
