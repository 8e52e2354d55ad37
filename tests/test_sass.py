"""SASS checks of the built sm_100a kernels (CPU only: cuobjdump on the in-tree objects).

They pin what the roofline claims rest on: K2's main loop is 32 DADD + 1
LDS.128 + sign-flip LOP3s per element with no spills, its diagonal stream uses the bulk-copy
(TMA) engine, and the run-pointer instantiation that keeps ptxas' fast schedule
(profiles/r01_k2_codegen.md) is the one with the 1198-instruction two-block loop."""
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT

OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_kernels.o")
SEG_OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_k2seg.o")
SHARE_OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_k2share.o")
C_OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_k2c.o")
CSEG_OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_k2cseg.o")
Q_OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_k2q.o")
WHT_OBJ = os.path.join(ROOT, "paper_2401_16378_b200", "csrc", "build", "pd_wht.o")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

pytestmark = pytest.mark.skipif(not (os.path.exists(OBJ) and os.path.exists(CUOBJDUMP)),
                                reason="kernels not built or cuobjdump missing")


def sass_of(obj, fun):
    out = subprocess.run([CUOBJDUMP, "-sass", "-fun", fun, obj], capture_output=True, text=True,
                         check=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    assert ins, f"no SASS for {fun}"
    return ins


def innermost_loop(ins, min_dadd=512):
    addr = {a: i for i, (a, _) in enumerate(ins)}
    best = None
    for i, (a, t) in enumerate(ins):
        if "BRA" not in t:
            continue
        m = re.search(r"0x([0-9a-f]+)", t.split("BRA", 1)[1])
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            body = [x[1] for x in ins[addr[tgt]:i + 1]]
            if sum(b.startswith("DADD") for b in body) >= min_dadd and (best is None or len(body) < len(best)):
                best = body
    assert best is not None, "no DADD loop found"
    return best


K2_FAST = "_ZN3pdb17gray_xmask_kernelILi4ELb0ELb0EEEvNS_8K2ParamsE"


def test_k2_main_loop_is_pure_fp64_adds():
    ins = sass_of(OBJ, K2_FAST)
    body = innermost_loop(ins)
    ops = [b.split()[0] for b in body]
    n_dadd = sum(o == "DADD" for o in ops)
    n_lds = sum(o.startswith("LDS.128") for o in ops)
    # two unrolled 16-element blocks: 32 elements x 32 accumulators
    assert n_dadd == 1024 and n_lds == 32, (n_dadd, n_lds)
    assert not any(o.startswith(("DMUL", "DFMA", "LDL", "STL")) for o in ops)
    # FP64-pipe share of the issue slots (the kernel is FP64-add bound: 2 pipe cycles per DADD)
    assert n_dadd / len(body) > 0.85, len(body)
    # the schedule measured at 485.8 ms (profiles/r01_k2_codegen.md)
    assert len(body) == 1198, len(body)


def test_k2_streams_diagonals_with_bulk_copies():
    ops = [t.split()[0] for _, t in sass_of(OBJ, K2_FAST)]
    assert any(o.startswith("UBLKCP") for o in ops), "no cp.async.bulk (TMA engine) in K2"
    assert any(o.startswith("SYNCS") for o in ops), "no mbarrier wait in K2"


def test_no_local_memory_in_hot_kernels():
    for obj in (OBJ, WHT_OBJ, SHARE_OBJ, C_OBJ, CSEG_OBJ, Q_OBJ):
        log = open(obj + ".ptxas.log").read()
        for m in re.finditer(r"Function properties for (\S+)\n\s*(\d+) bytes stack frame, (\d+) bytes spill stores",
                             log):
            name, stack, spills = m.group(1), int(m.group(2)), int(m.group(3))
            if "gray_" in name or "wht_" in name or "diag_gather" in name:
                assert spills == 0 and stack == 0, (name, stack, spills)


def test_k2_segment_instantiation_is_separate_and_clean():
    """The host pipeline's walk-segment K2 is compiled alone (pd_k2seg.cu, ptxas -O1) so it
    cannot move the whole-walk kernel's schedule; it must still be the pure-DADD loop."""
    seg = "_ZN3pdb17gray_xmask_kernelILi4ELb1ELb0EEEvNS_8K2ParamsE"
    listing = subprocess.run([CUOBJDUMP, "-sass", OBJ], capture_output=True, text=True).stdout
    assert seg not in listing, "segment instantiation leaked into pd_kernels.o"
    body = innermost_loop(sass_of(SEG_OBJ, seg))
    ops = [b.split()[0] for b in body]
    assert sum(o == "DADD" for o in ops) == 1024
    assert not any(o.startswith(("LDL", "STL")) for o in ops)


def dadd_loops(ins):
    """DADD count of every backward-branch loop body with at least 32 DADDs"""
    addr = {a: i for i, (a, _) in enumerate(ins)}
    out = {}
    for i, (a, t) in enumerate(ins):
        if "BRA" not in t:
            continue
        m = re.search(r"0x([0-9a-f]+)", t.split("BRA", 1)[1])
        if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
            body = [x[1] for x in ins[addr[int(m.group(1), 16)]:i + 1]]
            n = sum(b.startswith("DADD") for b in body)
            if n >= 32 and (n not in out or len(body) < len(out[n])):
                out[n] = body
    return out


def share_kernels():
    syms = subprocess.run([CUOBJDUMP, "-symbols", SHARE_OBJ], capture_output=True, text=True).stdout
    names = sorted(set(re.findall(r"(_Z\S*gray_share_kernelILb[01]EE\S*)", syms)))
    assert len(names) == 2, names
    return names


@pytest.mark.skipif(not os.path.exists(SHARE_OBJ), reason="K2s not built")
def test_k2s_has_one_pure_dadd_loop_per_live_chain_count():
    """K2s (pd_k2share.cu): one loop body per live-chain count (1, 2, 4, 8, 16 chains x re/im x
    32 elements = 64 ... 1024 DADDs), the 16-chain one with K2's instruction mix, and no
    multiplies or local memory anywhere in the loops."""
    for fun in share_kernels():
        loops = dadd_loops(sass_of(SHARE_OBJ, fun))
        for n in (64, 128, 256, 512, 1024):
            assert n in loops, (fun, sorted(loops))
            ops = [b.split()[0] for b in loops[n]]
            assert not any(o.startswith(("DMUL", "DFMA", "LDL", "STL")) for o in ops)
            assert sum(o.startswith("LDS") for o in ops) == 32
        assert 1024 / len(loops[1024]) > 0.85, len(loops[1024])


@pytest.mark.skipif(not os.path.exists(CSEG_OBJ), reason="K2s-c not built")
def test_k2s_c_has_sixteen_zlo_bodies_with_k2_loops():
    """K2s-c (N >= 13): one body per compile-time ZLO (16), each with the five live-chain loops;
    the element signs are DADD operand modifiers, so the 16-chain loop has K2's mix (1024 DADD,
    32 LDS.128, no 3-input sign-word LOP3) and there are no multiplies or local memory."""
    found = []
    for obj in (C_OBJ, CSEG_OBJ):  # one instantiation per translation unit
        syms = subprocess.run([CUOBJDUMP, "-symbols", obj], capture_output=True, text=True).stdout
        names = sorted(set(re.findall(r"(_Z\S*gray_share_c_kernelILb[01]EE\S*)", syms)))
        assert len(names) == 1, (obj, names)
        found.append((obj, names[0]))
    for obj, fun in found:
        ins = sass_of(obj, fun)
        addr = {a: i for i, (a, _) in enumerate(ins)}
        hot = []
        for i, (a, t) in enumerate(ins):
            m = re.search(r"0x([0-9a-f]+)", t.split("BRA", 1)[1]) if "BRA" in t else None
            if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
                body = [x[1] for x in ins[addr[int(m.group(1), 16)]:i + 1]]
                if sum(b.startswith("DADD") for b in body) == 1024:
                    hot.append(body)
        assert len(hot) == 16, (fun, len(hot))
        for body in hot:
            ops = [b.split()[0] for b in body]
            assert sum(o.startswith("LDS") for o in ops) == 32
            assert not any(o.startswith(("DMUL", "DFMA", "LDL", "STL")) for o in ops)
            assert not any(b.startswith("LOP3") and "0x96" in b for b in body)
            assert len(body) <= 1210, len(body)
