"""Per-kernel durations of an ncu launch list (`--metrics
gpu__time_duration.sum --csv`), in launch order, with the sum per
operator step (K1 -> K3 -> K4 triples) -- the kernel-time side of the
bench's CUDA-event step time.  python tools/launch_sum.py launches.csv"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                unit = d["Metric Unit"]
                v = float(d["Metric Value"]) * {"nsecond": 1e-3, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
                out.append((d["Kernel Name"].split("(")[0].replace("void ", ""), v, d["Grid Size"]))
    return out


def main():
    ks = [k for k in load(sys.argv[1]) if any(t in k[0] for t in ("r2c", "c2r", "cgemm"))]
    for i, (name, us, grid) in enumerate(ks):
        print(f"{i:3d} {name:40s} {us:8.2f} us  grid {grid}")
    agg = collections.defaultdict(list)
    for name, us, _ in ks:
        agg[name].append(us)
    for name, v in agg.items():
        print(f"{name:40s} n={len(v):3d} mean {sum(v) / len(v):8.2f} us")
    # op triples: sum of each consecutive (r2c, gemm, c2r)
    trip = [ks[i:i + 3] for i in range(0, len(ks) - 2, 3) if "r2c" in ks[i][0]]
    sums = [sum(k[1] for k in t) for t in trip]
    if len(sums) >= 3:
        print("per-op kernel sums (us):", [round(x, 1) for x in sums])
        print("last fprop+bprop+accGrad step kernel sum (us): %.1f" % sum(sums[-3:]))


if __name__ == "__main__":
    main()
