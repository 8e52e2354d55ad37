import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2401_16378_b200 as pd
dev = torch.device("cuda:0")
for nq in (12, 14):
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=dev)
    pd.device.random_matrix(nq, 3, g.data_ptr(), 0)
    c = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    scr = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    pd.device.decompose(nq, g.data_ptr(), c.data_ptr(), scr.data_ptr(), "wht", 0)
    g2 = torch.empty_like(g)
    f = lambda: pd.device.recompose(nq, c.data_ptr(), g2.data_ptr(), scr.data_ptr(), 0)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(5)]; b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    err = float(torch.max(torch.abs(g2 - g)))
    print(f"N={nq}: recompose {ms:.3f} ms = {32*4**nq/ms/1e6:.0f} GB/s algorithmic, max|G'-G| = {err:.2e}")
