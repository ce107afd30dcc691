#!/bin/bash
# ncu --set full of the standalone operators at configs[2] (32^3 p9 deformed, 32.8M DOF: HBM-bound):
# nb_ax (local, k_ax), nb_dssum structured (k_dssum_rows) and CSR (k_gs, NB_DSSUM=csr).
# Run on the GPU box; summarise here with python tools/ncu_summary.py gpurun_out/r2/ops_<pol>.ncu-rep
set -e
out=gpurun_out/r2
mkdir -p $out
for pol in ${@:-mixed fp64}; do
  python tools/bench_ops.py --cases 32x32x32p9d --policies $pol --reps 2 > $out/ops_plain_$pol.log 2>&1
  ncu --set full --clock-control none --import-source on -k "regex:k_ax|k_dssum_rows" -s 1 -c 4 -f -o $out/ops_$pol \
      python tools/bench_ops.py --cases 32x32x32p9d --policies $pol --reps 1 > $out/ops_ncu_$pol.log 2>&1
  NB_DSSUM=csr ncu --set full --clock-control none -k "regex:k_gs<" -c 2 -f -o $out/ops_csr_$pol \
      python tools/bench_ops.py --cases 32x32x32p9d --policies $pol --reps 1 > $out/ops_ncu_csr_$pol.log 2>&1
done
