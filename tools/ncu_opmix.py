"""Executed-instruction mix (by SASS opcode) of one kernel in an ncu report.

  python tools/ncu_opmix.py report.ncu-rep <kernel-regex>
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    iE, iSrc = h.index("Instructions Executed"), h.index("Source")
    c = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(h) or not (r[iE] or "0").isdigit():
            continue
        ins = r[iSrc].split()
        if not ins:
            continue
        op = ins[1] if ins[0].startswith("@") else ins[0]
        c[op.split(".")[0]] += int(r[iE] or 0)
    tot = sum(c.values())
    print("total warp-instructions", tot)
    for k, v in c.most_common(30):
        print(f"{k:10s} {v:10d} {v / tot:.3f}")


if __name__ == "__main__":
    main()
