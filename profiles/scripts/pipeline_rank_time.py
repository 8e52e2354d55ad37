"""Device time of one rank's share of the pipelined NCCL mode, measured alone on one GPU.

The transfers are replaced by instantly available data (recv: a device copy of the right size,
prepared beforehand; send: nothing), so the number is the rank's kernel time inside the
pipeline schedule (rank 0: K1 of every rank's blocks and the unpacking of the gathered runs;
every rank: the per-block walks and the run packing) — what the NCCL transfers must hide
behind. Usage:
    python profiles/scripts/pipeline_rank_time.py [N] [P] [block sizes, e.g. 256,256,512,...]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_16378_b200 as pd  # noqa: E402
from paper_2401_16378_b200.sharding import NcclPipeline, ShardPlan  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 14
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
SIZES = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 and sys.argv[3] != "-" else None
dev = torch.device("cuda:0")
G = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=dev)
pd.device.random_matrix(nq, 7, G.data_ptr(), 0)


class Instant:
    """recv: copy a prepared piece of the same size on the current stream; send: nothing"""

    def __init__(self, pieces):
        self.pieces = pieces

    def exchange(self, ops_list):
        for kind, t, peer in ops_list:
            if kind == "recv":
                t.copy_(self.pieces[t.numel()])


for rank in (0, P - 1):
    plan = ShardPlan(nq, P, rank)
    pipe = NcclPipeline(plan, dev, sizes=SIZES)
    needed = {sz << nq for _, sz in pipe.blocks} | {m[2] for m in pipe.meta}
    pipe.transport = Instant({n: torch.zeros(n, dtype=torch.complex128, device=dev) for n in needed})
    out = torch.empty(4**nq, dtype=torch.complex128, device=dev) if rank == 0 else None
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            pipe(G, out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(5):
            pipe(G, out)
        b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"N={nq} P={P} rank {rank}: {ms:.2f} ms per step, blocks {[sz for _, sz in pipe.blocks]}",
          flush=True)
    del pipe, out
    torch.cuda.empty_cache()
