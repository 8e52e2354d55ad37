"""A/B of K2s codegen variants: for each libpd_b200.so given, one device-resident N=14
decomposition (K1 + K2s, Gray path) timed 4x after 1 warm-up, plus a hash of all coefficient
bits (variants must equal the shipped build bit for bit). Each library runs in its own process."""
import hashlib, os, subprocess, sys

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    import ctypes, torch
    lib = ctypes.CDLL(sys.argv[2])
    N = int(os.environ.get("PD_N", "14"))
    g = torch.empty(4**N, dtype=torch.complex128, device="cuda:0")
    out = torch.empty_like(g); scr = torch.empty_like(g)
    vp = ctypes.c_void_p
    lib.pd_random_matrix_device.argtypes = [ctypes.c_uint, ctypes.c_uint64, vp, vp]
    lib.pd_decompose_device.argtypes = [ctypes.c_uint, vp, vp, vp, ctypes.c_int, vp]
    s = torch.cuda.current_stream().cuda_stream
    assert lib.pd_random_matrix_device(N, 1234, g.data_ptr(), s) == 0
    assert lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 0, s) == 0
    torch.cuda.synchronize()
    h = hashlib.sha1(out.view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:12]
    ts = []
    for _ in range(4):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); lib.pd_decompose_device(N, g.data_ptr(), out.data_ptr(), scr.data_ptr(), 0, s); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{os.path.basename(sys.argv[2]):28s} N={N} hash={h} ms={' '.join('%.2f' % t for t in ts)} min={min(ts):.2f}", flush=True)
else:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, "--one", lib], check=False)
