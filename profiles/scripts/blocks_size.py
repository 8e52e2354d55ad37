"""Per-launch size effect on the Gray kernel: pd_decompose_device_blocked with scratch for
blocks of B X-masks (sequential launches, one stream), N=14, against one launch."""
import ctypes, sys, torch
lib = ctypes.CDLL(sys.argv[1])
N = 14
g = torch.empty(4**N, dtype=torch.complex128, device="cuda:0")
out = torch.empty_like(g)
vp = ctypes.c_void_p
lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, vp, vp]
lib.pd_decompose_device_blocked.argtypes = [ctypes.c_uint, vp, vp, vp, ctypes.c_size_t, ctypes.c_int, vp]
assert lib.pd_random_matrix_device(N, 1234, g.data_ptr(), None) == 0
s = torch.cuda.current_stream().cuda_stream
for B in (16384, 8192, 4096, 2048, 1024, 512):
    scr = torch.empty(B * 2**N, dtype=torch.complex128, device="cuda:0")
    nb = scr.numel() * 16
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); rc = lib.pd_decompose_device_blocked(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), nb, 0, s); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b)); assert rc == 0, rc
    print(f"block {B:6d} X-masks: {min(ts):.2f} ms", flush=True)
    del scr
