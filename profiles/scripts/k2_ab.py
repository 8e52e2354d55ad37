"""A/B timing of K1+K2 (pd_decompose_device, Gray path) for a given libpd_b200.so."""
import ctypes, sys, torch
lib = ctypes.CDLL(sys.argv[1])
import os
N = int(os.environ.get("PD_N", "14"))
dev = torch.device("cuda:0")
g = torch.empty(4**N, dtype=torch.complex128, device=dev)
out = torch.empty_like(g); scr = torch.empty_like(g)
vp = ctypes.c_void_p
lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, vp, vp]
lib.pd_decompose_device.argtypes = [ctypes.c_uint, vp, vp, vp, ctypes.c_int, vp]
s = torch.cuda.current_stream().cuda_stream
assert lib.pd_random_matrix_device(N, 1234, g.data_ptr(), s) == 0
for _ in range(2):
    lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 0, s)
torch.cuda.synchronize()
ts = []
for _ in range(4):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 0, s); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(sys.argv[1], ["%.1f" % t for t in ts])
