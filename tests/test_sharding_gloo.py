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
