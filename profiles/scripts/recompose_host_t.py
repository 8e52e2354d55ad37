"""Python recompose on plain numpy arrays at N=12/14: wall time per call and round-trip error."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2401_16378_b200 as pd
for nq in (12, 14):
    d = 2**nq
    G = torch.empty((d, d), dtype=torch.complex128, device='cuda'); pd.device.random_matrix(nq, 3, G.data_ptr(), 0)
    g = G.cpu().numpy(); del G; torch.cuda.empty_cache()
    c = pd.decompose(g)
    for _ in range(3):
        t0 = time.perf_counter(); back = pd.recompose(c); t1 = time.perf_counter()
        print(f"N={nq} recompose(numpy) {1e3*(t1-t0):.1f} ms shape={back.shape} c_contig={back.flags.c_contiguous} writeable={back.flags.writeable} max|G'-G|={np.max(np.abs(back-g)):.2e}", flush=True)
        del back
