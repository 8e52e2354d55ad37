"""Device time: one K2s launch over all X-masks vs 32 block launches alternating two streams."""
import ctypes, sys, torch
lib = ctypes.CDLL(sys.argv[1])
N = 14
dim = 2**N
vp = ctypes.c_void_p
lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, vp, vp]
lib.pd_diag_gather_device.argtypes = [ctypes.c_uint, vp, ctypes.c_uint64, ctypes.c_uint64, vp, vp]
lib.pd_xmask_coeffs_device.argtypes = [ctypes.c_uint, vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint, vp, ctypes.c_int, ctypes.c_int, vp]
g = torch.empty(4**N, dtype=torch.complex128, device="cuda")
out = torch.empty_like(g); diag = torch.empty_like(g)
s0 = torch.cuda.current_stream()
assert lib.pd_random_matrix_device(N, 1234, g.data_ptr(), s0.cuda_stream) == 0
assert lib.pd_diag_gather_device(N, g.data_ptr(), 0, dim, diag.data_ptr(), s0.cuda_stream) == 0
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def whole():
    assert lib.pd_xmask_coeffs_device(N, diag.data_ptr(), 0, dim, 0, out.data_ptr(), 0, 0, s0.cuda_stream) == 0
def blocks(nb):
    ev = torch.cuda.Event(); ev.record(s0)
    sa.wait_event(ev); sb.wait_event(ev)
    xc = dim // nb
    for q in range(nb):
        s = sa if q & 1 else sb
        assert lib.pd_xmask_coeffs_device(N, diag.data_ptr() + q * xc * dim * 16, q * xc, xc, 0, out.data_ptr(), 0, 0, s.cuda_stream) == 0
    e1 = torch.cuda.Event(); e1.record(sa); e2 = torch.cuda.Event(); e2.record(sb)
    s0.wait_event(e1); s0.wait_event(e2)
for name, f in (("whole", whole), ("32 blocks", lambda: blocks(32)), ("8 blocks", lambda: blocks(8)), ("whole", whole)):
    f(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s0); f(); b.record(s0); torch.cuda.synchronize()
    print(name, "%.2f ms" % a.elapsed_time(b))
