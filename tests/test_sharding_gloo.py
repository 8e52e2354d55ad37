"""The multi-GPU sharding layer's host logic over real torch.distributed collectives
(gloo, world sizes 2 and 4, CPU processes): X-mask partition, broadcast of G, run
addressing and the grouped send/recv gather into rank 0's reference-ordered array (NCCL
mode), and the handle publication, mapping cache and barrier ordering of the peer mode, with
shared file mappings standing in for CUDA IPC.

The device compute is replaced by a CPU stand-in built on the oracle (tests only), so the
assembled output must equal the oracle's full decomposition value for value."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compute(N, G, x0, x_count, run_bits, dst, layout, diag):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    nq = N
    g = G.reshape(2**nq, 2**nq).numpy()
    low = 2 * (nq - run_bits)
    z = np.arange(2**nq, dtype=np.uint64)
    for x in range(x0, x0 + x_count):
        ns = O.xz_to_n(np.uint64(x), z, nq)
        vals = O.port().coeff_batch(g, ns, threads=1)
        if layout == "global":
            dst[torch.from_numpy(ns.astype(np.int64))] = torch.from_numpy(vals)
            continue
        # packed runs: run r (Z-mask top bits) at r * 4^(N-p), n's low 2(N-p) bits inside it
        rsel = (z >> np.uint64(nq - run_bits)).astype(np.int64)
        local = (ns & np.uint64((1 << low) - 1)).astype(np.int64)
        dst[torch.from_numpy((rsel << low) | local)] = torch.from_numpy(vals)


class _FileMapper:
    """CPU stand-in for CUDA IPC: rank 0's buffers live in shared file mappings, a handle is
    (path, element count), and opening maps the same file (MAP_SHARED)."""

    def __init__(self, tmpdir):
        self.tmpdir = tmpdir
        self.paths = {}

    def alloc(self, name, shape):
        path = os.path.join(self.tmpdir, name)
        n = int(np.prod(shape))
        t = torch.from_file(path, shared=True, size=n, dtype=torch.complex128).view(*shape)
        self.paths[t.data_ptr()] = (path, n)
        return t

    def export(self, buf):
        return self.paths[buf.data_ptr()]

    def open(self, handle):
        path, n = handle
        return torch.from_file(path, shared=True, size=n, dtype=torch.complex128)

    def close(self, mapped):
        pass

    def fence(self):
        pass


def _worker(rank, world, port, nq, result_path, mode="nccl"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_16378_b200.sharding import ShardedDecomposer
    from oracle import oracle as O
    dim = 2**nq
    mapper = _FileMapper(os.path.dirname(result_path)) if mode == "peer" else None
    if rank == 0:
        g0 = torch.from_numpy(O.port().random_matrix(nq, 4242))
        if mapper:
            G = mapper.alloc("G.bin", (dim, dim))
            G.copy_(g0)
            out = mapper.alloc("out.bin", (4**nq,))
            out.zero_()
        else:
            G, out = g0, torch.zeros(4**nq, dtype=torch.complex128)
    else:
        G = torch.zeros((dim, dim), dtype=torch.complex128)  # filled by the broadcast (nccl mode)
        out = None
    sd = ShardedDecomposer(nq, torch.device("cpu"), compute=_oracle_compute, mode=mode,
                           mapper=mapper)
    assert sd.plan.x_count == dim // world and sd.plan.x0 == rank * dim // world
    for _ in range(2):  # the second step reuses the cached peer mappings
        sd(G, out)
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["nccl", "peer"])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gather_matches_oracle(tmp_path, world, mode):
    nq = 5
    result = str(tmp_path / "out.npy")
    mp.start_processes(_worker, args=(world, _free_port(), nq, result, mode), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(result)
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    want = O.port().decompose(O.port().random_matrix(nq, 4242))
    assert np.all(got == want)


def test_plan_rejects_bad_world_sizes():
    from paper_2401_16378_b200.sharding import ShardPlan
    with pytest.raises(ValueError):
        ShardPlan(5, 3, 0)
    with pytest.raises(ValueError):
        ShardPlan(2, 8, 0)
    p = ShardPlan(6, 8, 5)
    assert (p.run_bits, p.x_count, p.x0, p.run_len) == (3, 8, 40, 64)
    assert sorted(o for g in range(8) for o in p.offsets(g)) == list(range(0, 4**6, 64))


# ---------------------------------------------------------------------------------------------
# the pipelined NCCL mode's schedule (sharding.NcclPipeline) with numpy stand-ins of its device
# primitives: which diagonal rows go to which rank in which order, the per-block walks in both
# output layouts and the block packing / unpacking of the runs. The stand-in walk sums in a
# different order (a matrix product), so results are compared to the oracle within 1e-12.

class CpuPipelineOps:
    """numpy restatements of the pipeline's device primitives (include/pd_api.h)"""

    def begin(self):
        pass

    def end(self):
        pass

    def on(self, name):
        import contextlib
        return contextlib.nullcontext()

    def record(self, name):
        return None

    def wait(self, name, ev):
        pass

    def gather(self, st, N, G, x0, x_count, out):  # K1: out[(x - x0) 2^N + i] = G[i ^ x][i]
        dim = 1 << N
        g = G.reshape(dim, dim).numpy()
        i = np.arange(dim, dtype=np.int64)[None, :]
        x = np.arange(x0, x0 + x_count, dtype=np.int64)[:, None]
        out.numpy()[:x_count * dim] = g[i ^ x, i].reshape(-1)

    def coeffs(self, st, N, diag, x0, x_count, run_bits, out, layout):
        from oracle import oracle as O
        dim = 1 << N
        ks = np.arange(dim, dtype=np.int64)
        gk = ks ^ (ks >> 1)
        z = np.arange(dim, dtype=np.int64)
        sign = 1.0 - 2.0 * (np.bitwise_count(gk[:, None] & z[None, :]) & 1)
        S = diag.numpy()[:x_count * dim].reshape(x_count, dim)[:, gk] @ sign
        o = out.numpy()
        low = 2 * (N - run_bits)
        for xl in range(x_count):
            x = x0 + xl
            ns = O.xz_to_n(np.uint64(x), z.astype(np.uint64), N).astype(np.int64)
            c = (-1j) ** np.bitwise_count(x & z) * S[xl] / dim
            if layout == "global":
                o[ns] = c
            else:
                o[((z >> (N - run_bits)) << low) | (ns & ((1 << low) - 1))] = c

    def copy_runs(self, st, src, dst, run_len, src_off, dst_off):
        for a, b in zip(src_off.tolist(), dst_off.tolist()):
            dst[b:b + run_len] = src[a:a + run_len]

    def offsets(self, values):
        return torch.tensor(values, dtype=torch.int64)


def _pipeline_worker(rank, world, port, nq, blocks, result_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_16378_b200.sharding import ShardedDecomposer
    from oracle import oracle as O
    dim = 2**nq
    if rank == 0:
        G = torch.from_numpy(O.port().random_matrix(nq, 4343))
        out = torch.full((4**nq,), complex(np.nan, np.nan), dtype=torch.complex128)
    else:
        G = torch.full((dim, dim), complex(np.nan, np.nan), dtype=torch.complex128)  # never read
        out = None
    sd = ShardedDecomposer(nq, torch.device("cpu"), mode="nccl", pipeline_ops=CpuPipelineOps(),
                           pipeline_blocks=blocks)
    assert sd.mode == "nccl" and sd.pipeline is not None
    for _ in range(2):
        sd(G, out)
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nq,blocks", [(2, 6, None), (4, 6, [2, 2, 4, 4, 2, 2]), (8, 7, None),
                                             (4, 8, [8, 8, 16, 16, 8, 8]), (2, 8, [128])])
def test_nccl_pipeline_schedule_matches_oracle(tmp_path, world, nq, blocks):
    result = str(tmp_path / "out.npy")
    mp.start_processes(_pipeline_worker, args=(world, _free_port(), nq, blocks, result),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(result)
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    want = O.port().decompose(O.port().random_matrix(nq, 4343))
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


def test_xmask_blocks_plans():
    from paper_2401_16378_b200.sharding import xmask_blocks
    assert xmask_blocks(2048) == [(0, 256), (256, 256), (512, 512), (1024, 512), (1536, 256), (1792, 256)]
    assert xmask_blocks(8192) == [(0, 2048), (2048, 2048), (4096, 2048), (6144, 2048)]
    assert xmask_blocks(512) == [(0, 256), (256, 256)]
    for B in (1, 2, 16, 64, 1024, 4096):
        blocks = xmask_blocks(B)
        assert sum(sz for _, sz in blocks) == B
        assert all(off % sz == 0 for off, sz in blocks)
    with pytest.raises(ValueError):
        xmask_blocks(64, [16, 32, 16])   # 32 at offset 16 is not aligned
    with pytest.raises(ValueError):
        xmask_blocks(64, [32])
