"""K2s kernel forms against each other, bit for bit, over the whole coefficient array.

The Gray path has four kernels that must agree exactly: K2 (PD_K2SHARE=0: every chain
computed in full), K2s with per-thread sign words (PD_K2S_C=0; N in [9, 12] always) and K2s-c,
whose CTAs share the low four Z-mask bits as a compile-time constant (N >= 13), and K2q for
the host pipeline's first walk segments (PD_K2Q=0 turns it off). The kernel choice is read
once per process, so each form runs in its own subprocess."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2401_16378_b200 as pd
nq, kind, path = int(sys.argv[2]), sys.argv[3], sys.argv[4]
d = 2 ** nq
rng = np.random.default_rng(900 + nq)
if kind == "normal":
    g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
elif kind == "band":      # 0/1 band: exact cancellations, exact zeros
    g = np.triu(np.tril(np.ones((d, d)), 2), -1).astype(complex)
else:                     # small integers: every partial sum exact
    g = (rng.integers(-3, 4, (d, d)) + 1j * rng.integers(-3, 4, (d, d))).astype(complex)
gd = torch.from_numpy(g).to("cuda:0")
out = torch.empty(4 ** nq, dtype=torch.complex128, device="cuda:0")
scr = torch.empty_like(out)
if path == "device":
    pd.device.decompose(nq, gd.data_ptr(), out.data_ptr(), scr.data_ptr(), "gray", 0)
    torch.cuda.synchronize()
    res = out.cpu().numpy()
else:                     # host buffers: the segmented pipeline (partial sums across launches)
    res = pd.decompose(g)
raw = hashlib.sha1(res.tobytes()).hexdigest()
canon = hashlib.sha1((res + 0.0).tobytes()).hexdigest()  # -0.0 -> +0.0: equal values, equal hash
print("HASH", raw, canon)
"""


def run(nq, kind, path, env):
    """(raw-bits hash, value hash) of one decomposition in a subprocess with `env` set"""
    e = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(nq), kind, path], env=e, check=True,
                       timeout=600, capture_output=True, text=True)
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("HASH ")][-1]
    return tuple(line.split()[1:])


@pytest.mark.parametrize("nq,kind", [(13, "normal"), (13, "band"), (13, "int"), (14, "band")])
def test_k2s_c_bitwise_equal_sign_word_form(cuda, nq, kind):
    u = run(nq, kind, "device", {})
    w = run(nq, kind, "device", {"PD_K2S_C": "0"})
    assert u[0] == w[0]  # same bits
    if nq <= 13:  # and K2 (full chains): equal values (an exact zero's sign may differ)
        k2 = run(nq, kind, "device", {"PD_K2SHARE": "0"})
        assert u[1] == k2[1]


@pytest.mark.parametrize("nq,kind", [(12, "normal"), (13, "normal"), (13, "band"), (14, "normal")])
def test_host_pipeline_segments_bitwise(cuda, nq, kind):
    """host buffers: walk segments that stop and restart mid-walk from stored raw sums — the
    first-half segments on K2q (4 and 2 Z-masks per thread), the rest on K2s — against one
    whole-walk launch of the sign-word kernel, and against the same pipeline without K2q"""
    u = run(nq, kind, "host", {})
    w = run(nq, kind, "device", {"PD_K2S_C": "0"})
    assert u[0] == w[0]
    if nq <= 13:
        assert u[0] == run(nq, kind, "host", {"PD_K2Q": "0"})[0]


@pytest.mark.parametrize("nq,kind,sb", [(13, "normal", "40"), (14, "normal", "64"), (14, "band", "80")])
def test_k2s_c_superblock_order_bitwise(cuda, nq, kind, sb):
    """PD_K2SC_SB: the traffic-lean X-mask superblock order of K2s-c (a partial last superblock
    at S = 40 and 80) computes every coefficient in the same order, so the bits are the same"""
    assert run(nq, kind, "device", {"PD_K2SC_SB": sb})[0] == run(nq, kind, "device", {})[0]
