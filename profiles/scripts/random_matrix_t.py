"""Python random_matrix(N, seed) (the reference generator on the GPU, into a new numpy array):
wall time per call at N=12/14 and agreement with the device-pointer form."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2401_16378_b200 as pd
for nq in (12, 14):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); a = pd.random_matrix(nq, 11); ts.append(time.perf_counter() - t0)
    G = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device='cuda')
    pd.device.random_matrix(nq, 11, G.data_ptr(), 0)
    same = np.array_equal(a.view(np.uint64), G.cpu().numpy().view(np.uint64))
    print(f"N={nq} random_matrix {' '.join('%.1f' % (1e3 * t) for t in ts)} ms, equal to device form: {same}", flush=True)
    del a, G
    torch.cuda.empty_cache()
