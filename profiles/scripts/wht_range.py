"""One WHT decomposition inside a cudaProfilerStart/Stop range (for ncu --replay-mode range)."""
import ctypes, sys, os, torch
lib = ctypes.CDLL(sys.argv[1])
N = int(os.environ.get("PD_N", "14"))
path = int(os.environ.get("PD_PATH", "1"))
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
for _ in range(2):
    assert lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), path, s) == 0
torch.cuda.synchronize()
torch.cuda.profiler.start()
assert lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), path, s) == 0
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
