"""Compile one translation unit with -Xptxas -v and print registers / spills per kernel.

  python tools/ptxas_regs.py nb_cg_mixed.cu [-DNB_FLATB=0 ...] [--filter k_cg_mega]
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2503_02134_b200", "csrc")


def main():
    args = sys.argv[1:]
    filt = None
    if "--filter" in args:
        i = args.index("--filter")
        filt = args[i + 1]
        del args[i:i + 2]
    unit, extra = args[0], args[1:]
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
           "-Xcompiler", "-fPIC", "-ftz=false", "-prec-div=true", "-prec-sqrt=true", f"-I{ROOT}/include",
           f"-I{CSRC}", "-Xptxas", "-v", "-c", "-o", "/tmp/ptxas_regs.o", os.path.join(CSRC, unit), *extra]
    out = subprocess.run(cmd, capture_output=True, text=True).stderr
    name = None
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
        if m:
            name = m.group(1)
        m2 = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m2 and name:
            spill = (m2.group(1), m2.group(2))
        m3 = re.search(r"Used (\d+) registers", line)
        if m3 and name:
            dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
            if not filt or filt in dem:
                print(f"{m3.group(1):>4} regs  spill st/ld {spill[0]}/{spill[1]}  {dem[:140]}")
            name = None


if __name__ == "__main__":
    main()
