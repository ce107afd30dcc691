#!/bin/bash
# ncu --set full of the Schwarz solveM kernel (k_sw_apply) at configs[2] (32^3 p9 deformed) and
# configs[1] (16^3 p7), mixed; summaries written on the box (reports too large to bring back)
set -u
tag=${1:-sw}; out=gpurun_out/r2; mkdir -p $out
export NB_NO_BUILD=1
for c in 32x32x32p9d 16x16x16p7; do
  ncu --set full --clock-control none --import-source on -k regex:k_sw_apply -s 1 -c 1 -f -o $out/${tag}_$c \
     python tools/schwarz_bench.py --apply --cases $c --policies mixed --reps 1 > $out/${tag}_$c.log 2>&1; echo "$c rc=$?"
done
for r in $out/${tag}_*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_report.py $r > $b.txt 2>&1
  ncu -i $r --page source --csv --print-source cuda,sass > $b.src.csv 2>/dev/null; gzip -f $b.src.csv
  rm -f $r
done
