"""Pageable-host costs at N=14 (4 GiB in, 4 GiB out): what the reference's normal caller (a plain
numpy array, bindings/module.cpp:21-33) pays through decompose(), and the building blocks of a
fix: cudaHostRegister/Unregister of a caller buffer, first-touch of a fresh output array,
multi-threaded host memcpy, pageable cudaMemcpy. Prints one line per measurement."""
import ctypes
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_16378_b200 as pd  # noqa: E402

N = int(os.environ.get("N", "14"))
dim = 1 << N
nbytes = 16 * dim * dim
cudart = torch.cuda.cudart()


def t(f, reps=1):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, r


print(f"N={N} bytes={nbytes} cores={os.cpu_count()} thp="
      f"{open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip()}", flush=True)
torch.cuda.init()
G = torch.empty(dim * dim * 2, dtype=torch.float64, device="cuda")
pd.device.random_matrix(N, 7, G.data_ptr(), 0)
torch.cuda.synchronize()
g = G.cpu().numpy().view(np.complex128).reshape(dim, dim)  # pageable, touched
del G
torch.cuda.empty_cache()

s, _ = t(lambda: np.empty(dim * dim, np.complex128))
print(f"np.empty                  {s*1e3:9.2f} ms", flush=True)
s, a = t(lambda: np.zeros(dim * dim, np.complex128))
print(f"np.zeros (lazy)           {s*1e3:9.2f} ms", flush=True)
s, _ = t(lambda: a.fill(0))
print(f"first touch 1 thread      {s*1e3:9.2f} ms  ({nbytes/s/1e9:.1f} GB/s)", flush=True)
del a


def touch_mt(arr, threads):
    flat = arr.view(np.uint8)
    per = (flat.size + threads - 1) // threads
    libc = ctypes.CDLL(None)
    libc.memset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
    base = flat.ctypes.data

    def run(k):
        lo, hi = k * per, min(flat.size, (k + 1) * per)
        if hi > lo:
            libc.memset(base + lo, 0, hi - lo)
    ths = [threading.Thread(target=run, args=(k,)) for k in range(threads)]
    [x.start() for x in ths]
    [x.join() for x in ths]


for th in (8, 16, 32):
    b = np.empty(dim * dim, np.complex128)
    s, _ = t(lambda: touch_mt(b, th))
    print(f"first touch {th:2d} threads    {s*1e3:9.2f} ms  ({nbytes/s/1e9:.1f} GB/s)", flush=True)
    s, _ = t(lambda: touch_mt(b, th))
    print(f"memset warm {th:2d} threads    {s*1e3:9.2f} ms  ({nbytes/s/1e9:.1f} GB/s)", flush=True)
    del b

out = np.empty(dim * dim, np.complex128)
touch_mt(out, 16)
for flags, name in ((0, "default"), (8, "readonly")):
    s, r = t(lambda: cudart.cudaHostRegister(g.ctypes.data, nbytes, flags))
    print(f"cudaHostRegister {name:8s} {s*1e3:9.2f} ms rc={r}", flush=True)
    s, r = t(lambda: cudart.cudaHostUnregister(g.ctypes.data))
    print(f"cudaHostUnregister        {s*1e3:9.2f} ms rc={r}", flush=True)
fresh = np.empty(dim * dim, np.complex128)
s, r = t(lambda: cudart.cudaHostRegister(fresh.ctypes.data, nbytes, 0))
print(f"cudaHostRegister fresh    {s*1e3:9.2f} ms rc={r}", flush=True)
cudart.cudaHostUnregister(fresh.ctypes.data)
del fresh

D = torch.empty(dim * dim * 2, dtype=torch.float64, device="cuda")
s, _ = t(lambda: D.copy_(torch.from_numpy(g.view(np.float64).reshape(-1))), reps=2)
print(f"H2D pageable torch        {s*1e3:9.2f} ms  ({nbytes/s/1e9:.1f} GB/s)", flush=True)
o64 = torch.from_numpy(out.view(np.float64))
s, _ = t(lambda: o64.copy_(D), reps=2)
print(f"D2H pageable torch        {s*1e3:9.2f} ms  ({nbytes/s/1e9:.1f} GB/s)", flush=True)
del D
torch.cuda.empty_cache()

pd.decompose(g, out=out)  # warm the context
for k in range(2):
    s, _ = t(lambda: pd.decompose(g, out=out))
    print(f"decompose(g, out=out) pageable, touched out  {s*1e3:9.2f} ms", flush=True)
for k in range(2):
    s, r = t(lambda: pd.decompose(g))
    del r
    print(f"decompose(g) pageable, fresh result          {s*1e3:9.2f} ms", flush=True)
pg = torch.empty(dim * dim * 2, dtype=torch.float64, pin_memory=True)
pg.copy_(torch.from_numpy(g.view(np.float64).reshape(-1)))
po = torch.empty(dim * dim * 2, dtype=torch.float64, pin_memory=True)
gp = pg.numpy().view(np.complex128).reshape(dim, dim)
opn = po.numpy().view(np.complex128)
for k in range(2):
    s, _ = t(lambda: pd.decompose(gp, out=opn))
    print(f"decompose pinned in/out                      {s*1e3:9.2f} ms", flush=True)
