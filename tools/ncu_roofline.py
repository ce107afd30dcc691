#!/usr/bin/env python3
"""Write profiles/r2_ncu_roofline.json + .txt from tools/ncu_roofline.sh captures (DRAM bytes per
CG iteration of the configs[2] megakernel launch, whole solve and each phase alone).

    python tools/ncu_roofline.py gpurun_out/r2 [--iterations 200] [--tag r2]
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3, "%": 1}


def metrics_csv(path):
    vals = {}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        v = float(row["Metric Value"].replace(",", ""))
        vals[row["Metric Name"]] = v * SCALE.get(row["Metric Unit"], 1)
    return vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dir")
    ap.add_argument("--iterations", type=int, default=200)
    ap.add_argument("--tag", default="r2")
    a = ap.parse_args()
    js, txt = {}, []
    for pol in ("mixed", "fp64", "fp32"):
        rep = os.path.join(a.dir, f"roof_{pol}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d = [r for r in ncu_summary.rows(rep) if "k_cg_mega" in r["kernel"]][0]
        tr = d["dram_rd"] + d["dram_wr"]
        rec = {"dram_bytes_per_iteration": tr / a.iterations, "kernel_us_under_ncu": d["us"],
               "dram_GBps_under_ncu": tr / (d["us"] * 1e-6) / 1e9, "dram_pct_of_peak_ncu": d.get("dram%"),
               "registers": d.get("regs"), "grid": d.get("grid"), "block": d.get("blk"),
               "source": f"profiles/{a.tag}_ncu_roofline.txt ({os.path.basename(rep)}: --set full, "
                         f"{a.iterations} iterations of configs[2], {d['kernel']})"}
        line = (f"{pol:6s} whole solve  {d['kernel'][:30]:30s} {d['us'] / 1e3:8.2f} ms  dram {tr / 1e9:8.3f} GB "
                f"({tr / a.iterations / 1e6:7.2f} MB/it)  {rec['dram_GBps_under_ncu']:6.0f} GB/s  "
                f"dram%={d.get('dram%', 0):5.1f} l1%={d.get('l1%', 0):5.1f} l2%={d.get('l2%', 0):5.1f} "
                f"occ%={d.get('occ%', 0):5.1f} regs={d.get('regs', 0):.0f} grid={d.get('grid', 0):.0f}x{d.get('blk', 0):.0f}")
        txt.append(line)
        for ph in ("A", "B"):
            f = os.path.join(a.dir, f"roof_{pol}_{ph}.csv")
            if not os.path.exists(f):
                continue
            m = metrics_csv(f)
            b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
            rec[f"phase{ph}_dram_bytes_per_iteration"] = b / a.iterations
            rec[f"phase{ph}_only_kernel_us_under_ncu"] = m["gpu__time_duration.sum"]
            rec[f"phase{ph}_only_dram_pct_ncu"] = m.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
            txt.append(f"{pol:6s} phase {ph} only {'':30s} {m['gpu__time_duration.sum'] / 1e3:8.2f} ms  dram "
                       f"{b / 1e9:8.3f} GB ({b / a.iterations / 1e6:7.2f} MB/it)  "
                       f"{b / (m['gpu__time_duration.sum'] * 1e-6) / 1e9:6.0f} GB/s  "
                       f"dram%={m.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}")
        js[f"configs2_{pol}"] = rec
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_roofline.json"), "w") as f:
        json.dump(js, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_roofline.txt"), "w") as f:
        f.write("# ncu (B200) of bench.py --roofline-only: configs[2] 32^3 p9 deformed, "
                f"{a.iterations} fixed CG iterations in one k_cg_mega launch (tools/ncu_roofline.sh)\n")
        f.write("# cold-cache and serialised under ncu: compare DRAM bytes and shares, not absolute times\n")
        f.write("\n".join(txt) + "\n")
    print("\n".join(txt))


if __name__ == "__main__":
    main()
