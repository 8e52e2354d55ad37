"""e2e timing of paper_2401_16378_b200.decompose on pinned host buffers (N=14)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2401_16378_b200 as pd
N = int(os.environ.get("PD_N", "14"))
path = os.environ.get("PD_PATHNAME", "gray")
g = torch.empty((2**N, 2**N), dtype=torch.complex128, device="cuda")
pd.device.random_matrix(N, 99, g.data_ptr(), 0)
gh = torch.empty(g.shape, dtype=torch.complex128, pin_memory=True); gh.copy_(g)
oh = torch.empty(4**N, dtype=torch.complex128, pin_memory=True)
a, b = gh.numpy(), oh.numpy()
pd.decompose(a, out=b, path=path)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); pd.decompose(a, out=b, path=path); ts.append((time.perf_counter() - t0) * 1e3)
print(os.environ.get("PD_E2E_SEGS"), os.environ.get("PD_E2E_BITS"), path, ["%.1f" % t for t in ts])
