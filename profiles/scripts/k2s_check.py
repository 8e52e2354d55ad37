"""K2s vs K2: bit-identical outputs (all coefficients) and timing, same process."""
import ctypes, sys, os, torch
lib = ctypes.CDLL(sys.argv[1])
N = int(os.environ.get("PD_N", "12"))
dev = torch.device("cuda:0")
g = torch.empty(4**N, dtype=torch.complex128, device=dev)
out = torch.empty_like(g); scr = torch.empty_like(g)
vp = ctypes.c_void_p
lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, vp, vp]
lib.pd_decompose_device.argtypes = [ctypes.c_uint, vp, vp, vp, ctypes.c_int, vp]
s = torch.cuda.current_stream().cuda_stream
assert lib.pd_random_matrix_device(N, 1234, g.data_ptr(), s) == 0
assert lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 0, s) == 0
torch.cuda.synchronize()
torch.save(out.view(torch.int64).cpu(), f"/tmp/k2_{os.environ.get('PD_K2SHARE','1')}_{N}.pt")
ts = []
for _ in range(3):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 0, s); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("N", N, "share", os.environ.get("PD_K2SHARE", "1"), ["%.2f" % t for t in ts])
