# Round-end measurement refresh (one gpurun call): bench line, slab-emulation bench line,
# launch list of the bench command, one ncu --set full capture of the configs[1] megakernel.
set -u
T=${TAG:-r1v20}
export NB_NO_BUILD=1
python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
python bench.py --mode slab --slabs 2 --quick --no-cpu > gpurun_out/bench_slab2_$T.json 2>&1; echo "slab rc=$?"
python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/bench_q_$T.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
      python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/ncu_launch_$T.log 2>&1; echo "launch rc=$?"
python tools/sweep.py --cases 16x16x16p7 --policies mixed --iters 587 --reps 1 > gpurun_out/sweep_q_$T.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:k_cg_mega -c 1 -o gpurun_out/prof_${T}_mega -f \
      python tools/sweep.py --cases 16x16x16p7 --policies mixed --iters 587 --reps 1 > gpurun_out/ncu_full_$T.log 2>&1; echo "full rc=$?"
