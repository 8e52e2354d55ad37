"""A/B of the pageable host path at N=14 (one process per variant, same box): wall time of
decompose(numpy g) -> new array, decompose(numpy g, out=touched numpy), and the pinned call.
Usage: python profiles/scripts/pageable_ab.py [N]   [thp,prefault;...]  (PD_RESULT_THP, PD_RESULT_PREFAULT)"""
import os
import subprocess
import sys

CHILD = r"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2401_16378_b200 as pd
N = int(sys.argv[1]); dim = 1 << N
G = torch.empty(dim * dim * 2, dtype=torch.float64, device='cuda')
pd.device.random_matrix(N, 7, G.data_ptr(), 0); torch.cuda.synchronize()
g = G.cpu().numpy().view(np.complex128).reshape(dim, dim); del G; torch.cuda.empty_cache()
out = np.ones(4**N, np.complex128)
def clock(f, reps=4):
    f(); t = []
    for _ in range(reps):
        t0 = time.perf_counter(); r = f(); t.append(time.perf_counter() - t0); del r
    return min(t) * 1e3, sorted(t)[len(t) // 2] * 1e3
pg = torch.empty(dim * dim, dtype=torch.complex128, pin_memory=True).numpy().reshape(dim, dim); pg[...] = g
po = torch.empty(4**N, dtype=torch.complex128, pin_memory=True).numpy()
for name, f in (("pinned in/out", lambda: pd.decompose(pg, out=po)),
                ("pageable, out=touched", lambda: pd.decompose(g, out=out)),
                ("pageable, fresh result", lambda: pd.decompose(g))):
    lo, med = clock(f)
    print(f"  {name:24s} min {lo:8.2f} ms  median {med:8.2f} ms", flush=True)
"""

N = sys.argv[1] if len(sys.argv) > 1 else "14"
VARIANTS = [v.split(",") for v in (sys.argv[2] if len(sys.argv) > 2 else "1,8;0,8;1,0;0,0").split(";")]
for thp, pf in VARIANTS:
    print(f"N={N} PD_RESULT_THP={thp} PD_RESULT_PREFAULT={pf} "
          f"PD_STAGE_WORKERS={os.environ.get('PD_STAGE_WORKERS', '-')}", flush=True)
    subprocess.run([sys.executable, "-c", CHILD, N],
                   env=dict(os.environ, PD_RESULT_THP=thp, PD_RESULT_PREFAULT=pf))
