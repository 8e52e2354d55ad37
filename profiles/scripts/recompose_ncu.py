"""One N=14 recompose (chunked inverse WHT passes) for ncu: run once to warm, then once under
the profiler's kernel filter. Usage under ncu: -k regex:wht_inv -s 40 -c 4"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2401_16378_b200 as pd
dev = torch.device("cuda:0")
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 14
g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=dev)
pd.device.random_matrix(nq, 3, g.data_ptr(), 0)
c = torch.empty(4**nq, dtype=torch.complex128, device=dev)
scr = torch.empty(4**nq, dtype=torch.complex128, device=dev)
pd.device.decompose(nq, g.data_ptr(), c.data_ptr(), scr.data_ptr(), "wht", 0)
g2 = torch.empty_like(g)
for _ in range(2):
    pd.device.recompose(nq, c.data_ptr(), g2.data_ptr(), scr.data_ptr(), 0)
torch.cuda.synchronize()
print("max|G'-G| =", float(torch.max(torch.abs(g2 - g))))
