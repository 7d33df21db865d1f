"""Opcode mix and stall samples of one kernel instance in an ncu report
(SASS source page): which instruction classes the warps issue and stall on.
  python tools/ncu_sass_mix.py report.ncu-rep <kernel-regex> [instance]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    inst = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    i0 = starts[inst]
    i1 = starts[inst + 1] - 1 if inst + 1 < len(starts) else len(rows)
    h = rows[i0]
    iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    body = [r for r in rows[i0 + 1:i1] if len(r) == len(h) and r[iS].isdigit()]
    by = collections.defaultdict(lambda: [0, 0])
    for r in body:
        op = r[iSrc].split()[0] if r[iSrc].split() else "?"
        if op.startswith("@"):
            op = r[iSrc].split()[1]
        op = op.split(".")[0]
        by[op][0] += int(r[iS])
        by[op][1] += int(r[iE] or 0)
    ts, te = sum(v[0] for v in by.values()), sum(v[1] for v in by.values())
    print(f"instance {inst}: {len(body)} SASS lines, {te} warp-instructions, {ts} stall samples")
    for op, (s_, e_) in sorted(by.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"  {op:10s} inst {e_:9d} ({100 * e_ / te:5.1f}%)  samples {s_:7d} ({100 * s_ / max(ts, 1):5.1f}%)")


if __name__ == "__main__":
    main()
