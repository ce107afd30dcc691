#!/usr/bin/env python3
"""Summarise an .ncu-rep (raw page) into one line per kernel launch: time, DRAM bytes,
throughputs, occupancy, registers.  Usage: python tools/ncu_summary.py rep.ncu-rep [--csv out.csv]"""
import csv
import io
import subprocess
import sys

M = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_rd"),
     ("dram__bytes_write.sum", "dram_wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
     ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
     ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
     ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "blk"),
     ("sm__cycles_active.avg", "sm_act_cyc"), ("gpc__cycles_elapsed.max", "cyc"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank_confl"),
     ("smsp__inst_executed.sum", "inst")]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {}
        for k, short in M:
            if k in hdr:
                i = hdr.index(k)
                v = row[i]
                u = units[i]
                if short == "kernel":
                    d[short] = v.split("(")[0].replace("void ", "").replace("nb::", "")
                    continue
                try:
                    f = float(v.replace(",", ""))
                except ValueError:
                    d[short] = v
                    continue
                if u == "Mbyte": f *= 1e6
                elif u == "Kbyte": f *= 1e3
                elif u == "Gbyte": f *= 1e9
                elif u == "ms" and short == "us": f *= 1e3
                elif u == "ns" and short == "us": f *= 1e-3
                elif u == "nsecond" and short == "us": f *= 1e-3
                elif u == "msecond" and short == "us": f *= 1e3
                d[short] = f
        res.append(d)
    return res


if __name__ == "__main__":
    rs = rows(sys.argv[1])
    for d in rs:
        t = d.get("us", 0)
        tr = (d.get("dram_rd", 0) + d.get("dram_wr", 0))
        print(f"{d['kernel'][:34]:34s} {t:7.2f}us dram {tr/1e6:7.2f}MB {tr/(t*1e-6)/1e9 if t else 0:7.0f}GB/s "
              f"dram%={d.get('dram%',0):5.1f} sm%={d.get('sm%',0):5.1f} l1%={d.get('l1%',0):5.1f} l2%={d.get('l2%',0):5.1f} "
              f"occ%={d.get('occ%',0):5.1f} regs={d.get('regs',0):.0f} grid={d.get('grid',0):.0f}x{d.get('blk',0):.0f} "
              f"act={d.get('sm_act_cyc',0)/max(d.get('cyc',1),1):.2f} bank={d.get('bank_confl',0):.0f}")
