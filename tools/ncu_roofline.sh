#!/bin/bash
# ncu evidence for bench.py's HBM roofline point (configs[2], 200 fixed iterations, one k_cg_mega
# launch): one --set full capture of the whole solve kernel per policy, and DRAM bytes of the same
# launch with only phase A / only phase B executed (NB_PHASE_ONLY, a measurement knob).
# Run on the GPU box:  bash tools/ncu_roofline.sh [policies...]   (default: mixed fp64)
# then here:            python tools/ncu_roofline.py gpurun_out/r2
set -e
out=gpurun_out/r2
mkdir -p $out
pols=${@:-mixed fp64}
for pol in $pols; do
  python bench.py --roofline-only --roof-policies $pol > $out/roof_plain_$pol.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_cg_mega -c 1 -f -o $out/roof_$pol \
      python bench.py --roofline-only --roof-policies $pol > $out/roof_ncu_$pol.log 2>&1
  for ph in A B; do
    NB_PHASE_ONLY=$ph ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
        --clock-control none -k regex:k_cg_mega -c 1 --csv --log-file $out/roof_${pol}_$ph.csv \
        python bench.py --roofline-only --roof-policies $pol > $out/roof_ncu_${pol}_$ph.log 2>&1
  done
done
