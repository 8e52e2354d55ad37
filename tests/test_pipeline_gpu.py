"""The pipelined NCCL mode's device data flow on one GPU (sharding.NcclPipeline).

Every rank of a P-rank run executes here as a host thread with its own streams and buffers on
the one GPU; the NCCL transfers are replaced by a loopback transport that hands a finished
buffer from one thread to another (the sender synchronises its stream first, so no kernel ever
waits on another rank's kernel). What runs on the device is exactly what each rank of a real
run executes: rank 0's K1 per X-mask block of every rank, the per-block walks (K2s / K2s-c and
the non-finite fixup) in both output layouts, and the run packing / unpacking. The assembled
output must equal the one-shot decomposition bit for bit.
"""
import queue
import threading

import numpy as np
import pytest

from conftest import device_scratch, same_or_both_nan

pytestmark = pytest.mark.gpu


class LoopbackTransport:
    def __init__(self, rank, queues):
        self.rank = rank
        self.q = queues

    def exchange(self, ops_list):
        import torch
        for kind, t, peer in ops_list:
            if kind == "send":
                c = t.clone()
                torch.cuda.current_stream().synchronize()
                self.q[(self.rank, peer)].put(c)
            else:
                src = self.q[(peer, self.rank)].get(timeout=600)
                t.copy_(src)
                # the sender's allocator may reuse src's memory once it is dropped: finish first
                torch.cuda.current_stream().synchronize()


def run_emulated(pd, nq, world, G, blocks=None):
    import torch
    from paper_2401_16378_b200.sharding import NcclPipeline, ShardPlan
    dev = G.device
    out = torch.full((4**nq,), complex(np.nan, np.nan), dtype=torch.complex128, device=dev)
    queues = {(a, b): queue.Queue() for a in range(world) for b in range(world)}
    pipes = [NcclPipeline(ShardPlan(nq, world, r), dev, sizes=blocks,
                          transport=LoopbackTransport(r, queues)) for r in range(world)]
    errors = []

    def rank_main(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                for _ in range(2):  # twice: buffers and streams are reused across steps
                    pipes[r](G, out if r == 0 else None)
                torch.cuda.current_stream().synchronize()
        except Exception as exc:  # pragma: no cover - reported below
            errors.append((r, repr(exc)))

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("nq,world", [(12, 8), (13, 4), (14, 2), (14, 8)])
def test_nccl_pipeline_dataflow_bit_exact(pd, cuda, nq, world):
    import torch
    G = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=cuda)
    pd.device.random_matrix(nq, pd.matrix_seed(20260823, nq, 0), G.data_ptr(), 0)
    want = torch.empty(4**nq, dtype=torch.complex128, device=cuda)
    scratch = device_scratch(pd, nq)
    pd.device.decompose(nq, G.data_ptr(), want.data_ptr(), scratch.data_ptr(), "gray", 0)
    del scratch
    out = run_emulated(pd, nq, world, G)
    assert torch.equal(out, want), (nq, world)


def test_nccl_pipeline_nonfinite_and_sub_blocks(pd, cuda, port):
    """an inf and a NaN on two ranks' diagonals: the final segments' fixup recomputes those
    X-masks with the reference's products, in both output layouts; several block plans"""
    import torch
    nq, world = 12, 4
    gh = port.random_matrix(nq, 1212)
    gh[5, 5 ^ 3000] = complex(np.inf, 0.25)    # X-mask 3000 (rank 2)
    gh[77, 77 ^ 100] = complex(0.5, np.nan)    # X-mask 100 (rank 0)
    G = torch.from_numpy(gh).to(cuda)
    from oracle import oracle as O
    ns = O.xmask_sample_indices(nq, [100, 3000])
    want_bad = port.coeff_batch(gh, ns)
    for blocks in (None, [1024], [256, 256, 512], [128, 128, 256, 256, 128, 128]):
        out = run_emulated(pd, nq, world, G, blocks=blocks).cpu().numpy()
        assert same_or_both_nan(out[ns.astype(np.int64)], want_bad), blocks
        ok = np.ones(4**nq, dtype=bool)
        ok[ns.astype(np.int64)] = False
        sample = np.flatnonzero(ok)[::997]
        assert same_or_both_nan(out[sample], port.coeff_batch(gh, sample.astype(np.uint64)))
