#!/bin/bash
# ncu --set full (with source) of phase A alone (NB_PHASE_ONLY=A) of the megakernel at 32^3 p9
# deformed, fp64 and mixed, 20 fixed iterations; plus the standalone k_ax and k_dssum_rows.
# Run on the GPU box: bash tools/ncu_phaseA.sh <out-tag> [lib]
set -u
tag=${1:-pa}; out=gpurun_out/r2; mkdir -p $out
export NB_NO_BUILD=1
[ -n "${2:-}" ] && export NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_$2.so
for pol in fp64 mixed; do
  NB_PHASE_ONLY=A ncu --set full --clock-control none --import-source on -k regex:k_cg_mega -c 1 -f -o $out/${tag}_A_$pol \
     python tools/sweep.py --cases 32x32x32p9d --policies $pol --iters 20 --reps 1 > $out/${tag}_A_$pol.log 2>&1; echo "A $pol rc=$?"
done
ncu --set full --clock-control none --import-source on -k "regex:k_ax|k_dssum_rows" -c 4 -f -o $out/${tag}_ops_mixed \
   python tools/bench_ops.py --cases 32x32x32p9d --policies mixed --reps 1 > $out/${tag}_ops.log 2>&1; echo "ops rc=$?"
# summaries on the box (the reports themselves are too large to bring back)
for r in $out/${tag}_*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_report.py $r > $b.txt 2>&1
  ncu -i $r --page source --csv --print-source cuda,sass > $b.src.csv 2>/dev/null; gzip -f $b.src.csv
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null; gzip -f $b.raw.csv
  [ -n "${KEEP_REP:-}" ] || rm -f $r
done
