"""Fixed memory (the reference's proj/tests/test_alloc.cpp promise, restated for the device
library): tests/fixed_memory.cpp counts every operator-new call of the process and the device's
free memory around 64 coeff_fast / coeff_slow calls (plain and MultCount forms) at N = 6, 10,
13 and around repeated full decompositions into a caller-owned array."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_coefficient_kernels_use_fixed_memory(tmp_path, pd, cuda):
    exe = str(tmp_path / "fixed_memory")
    libdir = os.path.join(ROOT, "paper_2401_16378_b200")
    cuda_home = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    "-I" + os.path.join(cuda_home, "include"), os.path.join(ROOT, "tests", "fixed_memory.cpp"),
                    "-L" + libdir, "-lpaulidecomp_b200", "-lpd_b200",
                    "-L" + os.path.join(cuda_home, "lib64"), "-lcudart",
                    "-Wl,-rpath," + libdir, "-Wl,-rpath," + os.path.join(cuda_home, "lib64"), "-o", exe],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
