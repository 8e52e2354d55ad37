"""Peer-memory sharding mode with real CUDA IPC (pd_ipc_export / pd_ipc_open): two rank
processes on one GPU, host plumbing over gloo.

Rank 1's K1 gathers its diagonals from rank 0's G through the mapped pointer and its K2 (or
fused WHT) stores the coefficients straight into rank 0's output; rank 0 then checks the array
against its own single-process decomposition. No kernel waits on another rank (the ordering is
two host barriers), so sharing one GPU between the ranks is safe (B200_PROFILING.md)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nq, path, result_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2401_16378_b200 as pd
    from paper_2401_16378_b200.sharding import ShardedDecomposer
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dim = 2**nq
    G = torch.empty((dim, dim), dtype=torch.complex128, device=dev)
    out = None
    if rank == 0:
        pd.device.random_matrix(nq, 777, G.data_ptr(), torch.cuda.current_stream().cuda_stream)
        out = torch.zeros(4**nq, dtype=torch.complex128, device=dev)
    sd = ShardedDecomposer(nq, dev, mode="peer", path=path)
    for _ in range(2):
        sd(G, out)
    ok = True
    if rank == 0:
        want = torch.empty_like(out)
        nb = pd.device.scratch_bytes(nq, 2**nq, path)
        scratch = torch.empty((nb + 15) // 16, dtype=torch.complex128, device=dev)
        pd.device.decompose(nq, G.data_ptr(), want.data_ptr(), scratch.data_ptr(), path,
                            torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        if path == "gray":
            ok = bool(torch.equal(out, want))
        else:
            ok = float(torch.max(torch.abs(out - want)) / torch.max(torch.abs(want))) <= 1e-11
        np.save(result_path, np.array([ok]))
    dist.barrier()
    sd.close_peers()
    dist.destroy_process_group()


@pytest.mark.parametrize("path", ["gray", "wht"])
def test_peer_mode_two_ranks_one_gpu(tmp_path, path):
    result = str(tmp_path / "ok.npy")
    mp.start_processes(_worker, args=(2, _free_port(), 10, path, result), nprocs=2, join=True,
                       start_method="spawn")
    assert bool(np.load(result)[0])
