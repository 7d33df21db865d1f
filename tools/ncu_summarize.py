"""Summarise ncu --set full reports into profiles/ (committed evidence).

  python tools/ncu_summarize.py <config> <report.ncu-rep> <out-prefix>

Writes <out-prefix>.json (per-launch metrics) and merges per-kernel DRAM
bytes per launch into profiles/ncu_summary.json (read by bench.py for the
roofline "traffic" field).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def kernel_key(name):
    m = re.search(r"(r2c_tma_kernel|c2r_tma_kernel|cgemm_bins_tcgen05|r2c_planes_kernel|c2r_planes_kernel|r2c128_cols_kernel|r2c128_rows_kernel|c2r128_rows_kernel|c2r128_cols_kernel)", name)
    return m.group(1) if m else name


def main():
    config, rep, prefix = sys.argv[1:4]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")]}
        for mname in METRICS:
            i = head.index(mname)
            v = float(r[i]) if r[i] not in ("", "n/a") else None
            u = units[i]
            if v is not None and mname.startswith("dram__bytes"):
                v *= SCALE.get(u, 1.0)  # -> MB
            if v is not None and mname == "gpu__time_duration.sum":
                v *= SCALE.get(u, 1.0)  # -> us
            d[mname] = v
        launches.append(d)
    with open(prefix + ".json", "w") as fh:
        json.dump({"report": os.path.basename(rep), "config": config,
                   "note": "ncu --set full --clock-control none; cold-cache serialised replay; "
                           "time in us, dram bytes in MB (writes still resident in L2 at kernel end "
                           "are not counted)", "launches": launches}, fh, indent=1)
    summ_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_summary.json")
    try:
        with open(summ_path) as fh:
            summ = json.load(fh)
    except Exception:
        summ = {}
    per = {}
    for d in launches:
        k = kernel_key(d["kernel"])
        b = (d["dram__bytes_read.sum"] or 0) + (d["dram__bytes_write.sum"] or 0)
        per.setdefault(k, []).append(b * 1e6)
    summ[config] = {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v),
                        "source": os.path.relpath(prefix + ".json", os.path.dirname(summ_path) + "/..")}
                    for k, v in per.items()}
    with open(summ_path, "w") as fh:
        json.dump(summ, fh, indent=1)
    print(json.dumps(summ[config], indent=1))


if __name__ == "__main__":
    main()
