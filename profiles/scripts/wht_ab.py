"""A/B timing of the WHT path (pd_decompose_device, path WHT) for a given libpd_b200.so."""
import ctypes, sys, os, torch
lib = ctypes.CDLL(sys.argv[1])
N = int(os.environ.get("PD_N", "14"))
dev = torch.device("cuda:0")
vp = ctypes.c_void_p
lib.pd_scratch_bytes.restype = ctypes.c_uint64
lib.pd_scratch_bytes.argtypes = [ctypes.c_uint, ctypes.c_uint64, ctypes.c_int]
g = torch.empty(4**N, dtype=torch.complex128, device=dev)
out = torch.empty_like(g)
scr = torch.empty((lib.pd_scratch_bytes(N, 2**N, 1) + 15) // 16, dtype=torch.complex128, device=dev)
lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, vp, vp]
lib.pd_decompose_device.argtypes = [ctypes.c_uint, vp, vp, vp, ctypes.c_int, vp]
s = torch.cuda.current_stream().cuda_stream
assert lib.pd_random_matrix_device(N, 1234, g.data_ptr(), s) == 0
for _ in range(3):
    assert lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 1, s) == 0
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 1, s); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(sys.argv[1], ["%.3f" % t for t in ts])
