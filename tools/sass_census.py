"""Per-kernel SASS opcode census of the product library: evidence that the
hot kernels are hand-written sm_100a tcgen05 / TMA code (UTCHMMA / UTCQMMA =
tcgen05.mma, UTMALDG / UTMASTG = TMA tensor load / store, UBLKCP = bulk
copy, LDTM / STTM = tcgen05.ld / st, UTCBAR = tcgen05.commit, SYNCS =
mbarrier).  python tools/sass_census.py [lib] > profiles/rNN_sass_census.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "UTCBAR",
       "SYNCS", "FFMA", "FADD", "FMUL", "LDS", "STS", "LDG", "STG"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1312_5851_b200", "lib",
                                                             "libfftconv_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", out)))
    kern = None
    counts = collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and kern:
            counts[kern][m.group(2)] += 1
    dem = {}
    names = list(counts)
    if names:
        d = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
        dem = dict(zip(names, d))
    print(f"# SASS census of {os.path.relpath(lib, ROOT)}  (cuobjdump -sass; arch {', '.join(arch)})")
    print("# static instruction counts per kernel (opcode families; not executed counts)")
    tot = collections.Counter()
    for k, c in counts.items():
        fam = collections.Counter()
        for op, n in c.items():
            fam[op.split(".")[0]] += n
        tot.update(fam)
        name = dem.get(k, k)
        if len(name) > 110:
            name = name[:107] + "..."
        print(f"\n{name}\n  total {sum(fam.values())}: " +
              ", ".join(f"{op} {fam[op]}" for op in KEY if fam[op]))
    print("\n# library total: " + ", ".join(f"{op} {tot[op]}" for op in KEY if tot[op]))


if __name__ == "__main__":
    main()
