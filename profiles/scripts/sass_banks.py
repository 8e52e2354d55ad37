"""Register-bank statistics of the hottest DADD loop in a cubin/object (offline, no GPU).

Usage: python sass_banks.py FILE.o|.so [kernel-substring]

For the loop body with the most DADDs (a backward branch target .. branch) it prints the
instruction mix and, for DADDs that read both source operands from the register file (neither
operand was marked .reuse by the previous DADD), how many pair registers in the same bank
(reg % 4, 64-bit pairs). The ncu source page of K2s showed those same-bank reads carry the
kernel's dispatch stalls (profiles/r01_k2s_banks.md)."""
import re
import subprocess
import sys
from collections import Counter


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.split("\n"):
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def hot_loop(ins):
    addr = {a: i for i, (a, _) in enumerate(ins)}
    best = None
    for i, (a, t) in enumerate(ins):
        if "BRA" not in t:
            continue
        m = re.search(r"0x([0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            nd = sum("DADD" in x for _, x in body)
            # innermost loop with the densest DADD mix
            if nd and (best is None or nd / len(body) > best[0] or (nd / len(body) == best[0] and len(body) < len(best[1]))):
                if nd >= 256:
                    best = (nd / len(body), body)
    return best[1] if best else []


def stats(body):
    c = Counter()
    prev = set()
    for _, x in body:
        m = re.match(r"DADD R(\d+), (-?)R(\d+)(\.reuse)?, (-?)R(\d+)(\.reuse)?", x)
        c["instr"] += 1
        if not m:
            if "LDS" in x:
                c["lds"] += 1
            prev = set()
            continue
        c["dadd"] += 1
        a, b = int(m.group(3)), int(m.group(6))
        ra, rb = ("A", a) not in prev, ("B", b) not in prev
        if ra and rb:
            c["both_read"] += 1
            if a % 4 == b % 4:
                c["same_bank"] += 1
        prev = set()
        if m.group(4):
            prev.add(("A", a))
        if m.group(7):
            prev.add(("B", b))
    return c


if __name__ == "__main__":
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 else "gray_share_kernelILb0"
    for name, ins in functions(path):
        if sub in name:
            c = stats(hot_loop(ins))
            print(f"{name[-60:]}: {dict(c)}")
