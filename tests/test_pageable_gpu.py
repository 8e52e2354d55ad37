"""Host buffers of every kind through the public API: pageable numpy arrays (the reference
binding's normal caller, bindings/module.cpp:21-33) go through the pinned slot rings of
csrc/pd_stage.cu, page-locked ones straight to DMA; every combination must give the bits the
device-resident decomposition gives."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, device_scratch, normal_matrix

pytestmark = pytest.mark.gpu


def device_result(pd, g, nq, path):
    import torch
    gd = torch.from_numpy(g).to("cuda:0")
    out = torch.empty(4**nq, dtype=torch.complex128, device="cuda:0")
    scratch = device_scratch(pd, nq, path="wht")
    pd.device.decompose(nq, gd.data_ptr(), out.data_ptr(), scratch.data_ptr(), path, 0)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def pinned_like(a):
    import torch
    t = torch.empty(a.size, dtype=torch.complex128, pin_memory=True)
    p = t.numpy().reshape(a.shape)
    p[...] = a
    return t, p


@pytest.mark.parametrize("path", ["gray", "wht"])
@pytest.mark.parametrize("nq", [9, 10, 12, 13])
def test_pageable_and_pinned_buffers_agree(pd, cuda, nq, path):
    g = normal_matrix(np.random.default_rng(4100 + nq), nq)
    want = device_result(pd, g, nq, path)
    keep_g, g_pin = pinned_like(g)
    keep_o, o_pin = pinned_like(np.zeros(4**nq, complex))
    o_page = np.full(4**nq, np.nan, complex)
    for src in (g, g_pin):
        assert np.array_equal(pd.decompose(src, path=path), want)  # fresh (pageable) result
        for dst in (o_page, o_pin):
            dst[...] = np.nan
            pd.decompose(src, path=path, out=dst)
            assert np.array_equal(dst, want)


def test_pageable_strided_input_is_coerced(pd, cuda, port):
    # a non-contiguous pageable view is copied by the binding (forcecast), then staged
    nq = 10
    big = normal_matrix(np.random.default_rng(77), nq + 1)
    g = big[::2, ::2]
    assert np.array_equal(pd.decompose(g), port.decompose(np.ascontiguousarray(g)))


SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2401_16378_b200 as pd
from conftest import normal_matrix
nq, path = {nq}, {path!r}
g = normal_matrix(np.random.default_rng(4200 + nq), nq)
np.save({dst!r}, pd.decompose(g, path=path))
"""


@pytest.mark.parametrize("path", ["gray", "wht"])
@pytest.mark.parametrize("nq", [11, 12])
def test_small_slots_and_few_workers(pd, cuda, tmp_path, nq, path):
    # 1 MiB slots and 3 workers: every upload band and download piece cycles the rings many
    # times over (N=12: 256 MiB each way through 4 + 16 slots)
    dst = str(tmp_path / "c.npy")
    env = dict(os.environ, PD_STAGE_SLOT_MB="1", PD_STAGE_WORKERS="3",
               PYTHONPATH=os.path.join(ROOT, "tests") + os.pathsep + ROOT)
    code = SCRIPT.format(root=ROOT, nq=nq, path=path, dst=dst)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    g = normal_matrix(np.random.default_rng(4200 + nq), nq)
    assert np.array_equal(np.load(dst), device_result(pd, g, nq, path))
