"""Top stall-sampled SASS lines of one kernel from an ncu report.

  python tools/ncu_hot.py report.ncu-rep <kernel-regex> [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
    h = rows[hi]
    iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[iS].isdigit()]
    tot = sum(int(r[iS]) for r in body)
    print("samples", tot, "warp-instructions", sum(int(r[iE] or 0) for r in body))
    for r in sorted(body, key=lambda r: -int(r[iS]))[:n]:
        print(f"{int(r[iS]):7d} {int(r[iE] or 0):9d}  {r[iSrc][:100]}")


if __name__ == "__main__":
    main()
