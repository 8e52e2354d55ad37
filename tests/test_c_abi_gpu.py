"""The C ABI from plain C (no C++, no Python in the process): examples/c_abi_demo.c."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_program_through_c_abi(tmp_path, pd):
    exe = str(tmp_path / "c_abi_demo")
    libdir = os.path.join(ROOT, "paper_2401_16378_b200")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L" + libdir, "-lpd_b200",
                    "-Wl,-rpath," + libdir, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.splitlines()[0] == "2.5+0i 2.5+0i 0-0.5i -1.5+0i"
    assert "out-of-range n -> -1" in r.stdout
