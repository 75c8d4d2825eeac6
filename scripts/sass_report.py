"""SASS evidence for profiles/ (no GPU needed): per-kernel instruction histograms of the built
libfblts.so (cuobjdump -sass) for the opcodes that show how the hot kernels work -- the bulk-copy
engine (UBLKCP), mbarriers (SYNCS), cp.async gathers (LDGSTS), fp64 math, warp shuffles -- and the
per-kernel resource usage (cuobjdump -res-usage: registers, shared memory, spills).

usage: python scripts/sass_report.py > profiles/r2_sass_report.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2405_10505_b200", "lib", "libfblts.so")
OPS = ["UBLKCP", "SYNCS", "LDGSTS", "LDGDEPBAR", "DEPBAR", "LDG", "STG", "LDS", "STS", "DFMA", "DADD", "DMUL",
       "MUFU", "SHFL", "BAR", "ATOM", "RED"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
        return out.split("\n")
    except (OSError, subprocess.CalledProcessError):
        return names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    hist = collections.OrderedDict()
    cur = None
    for line in sass.split("\n"):
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            hist[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            hist[cur][m.group(2)] += 1
    names = demangle(list(hist))
    print(f"# SASS opcode histograms of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass, static counts)")
    print("# kernel | " + " ".join(f"{o:>7s}" for o in OPS))
    for (k, h), n in sorted(zip(hist.items(), names), key=lambda t: t[1]):
        if not any(w in n for w in ("k_stage_tiled<6", "k_slow", "k_fine_s3<6", "k_fine_vel", "k_diag", "k_fine_sub<6",
                                    "k_coarse_vel", "k_rk4_stage<6", "k_vort")):
            continue
        short = re.sub(r"\(.*", "", n).replace("fblts::", "")
        print(f"{short[:34]:34s} | " + " ".join(f"{h.get(o, 0):7d}" for o in OPS))
    print()
    print("# resource usage (cuobjdump -res-usage)")
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True, check=True).stdout
    lines = res.split("\n")
    for i, line in enumerate(lines):
        m = re.match(r"\s*Function (\S+):", line)
        if m and i + 1 < len(lines):
            n = demangle([m.group(1)])[0]
            if any(w in n for w in ("k_stage_tiled<6", "k_slow_edge<10, false, false>", "k_slow_pre<6>", "k_fine_s3<6",
                                    "k_diag", "k_fine_vel")):
                print(f"{re.sub(r'[(].*', '', n).replace('fblts::', '')[:40]:40s} {lines[i + 1].strip()}")


if __name__ == "__main__":
    sys.exit(main())
