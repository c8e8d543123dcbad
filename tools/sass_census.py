"""Per-kernel SASS instruction census of the built product library (cuobjdump -sass):
the Blackwell-native evidence (UTCHMMA = tcgen05.mma, UTMALDG/UTMASTG = TMA tensor
load/store, UBLKCP = bulk copy, LDTM = tcgen05.ld, SYNCS = mbarrier ops) next to the
legacy forms (HMMA = mma.sync, LDGSTS = cp.async) and the FP32 arithmetic
(FFMA / FFMA2 / FMUL2) and shared loads (LDS).

    python tools/sass_census.py [lib] > profiles/r2_sass_census.txt
"""
import collections
import os
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "SYNCS", "HMMA", "LDGSTS", "FFMA2", "FMUL2", "FFMA",
       "DFMA", "LDS", "LDG", "STG"]


def census(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kern = None
    counts = collections.OrderedDict()
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9]+)(\.[\w.]+)?", line)
        if kern and m:
            counts[kern][m.group(2)] += 1
    return counts


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return out.splitlines()
    except OSError:
        return names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "paper_2006_06823_b200", "liblddmm_cuda.so")
    counts = census(lib)
    names = list(counts)
    pretty = demangle(names)
    print(f"# SASS census of {os.path.basename(lib)} (cuobjdump -sass, static instruction counts per kernel)")
    print("kernel | " + " | ".join(OPS))
    for n, p in sorted(zip(names, pretty), key=lambda t: t[1]):
        c = counts[n]
        if not any(c[o] for o in OPS):
            continue
        short = re.sub(r"\(.*", "", p.replace("(anonymous namespace)::", "")).replace("lddmm_b200::", "")
        print(f"{short[:90]} | " + " | ".join(str(c[o]) for o in OPS))


if __name__ == "__main__":
    main()
