# A/B of one library build under two environment settings (same session, interleaved)
export NB_NO_BUILD=1
for rep in 1 2; do
  for v in a b; do
    if [ $v = a ]; then env $AB_ENV_A python tools/sweep.py --cases $AB_CASES --policies $AB_POL --iters 200 --reps 5 > gpurun_out/abe_${rep}_$v.log 2>&1
    else env $AB_ENV_B python tools/sweep.py --cases $AB_CASES --policies $AB_POL --iters 200 --reps 5 > gpurun_out/abe_${rep}_$v.log 2>&1; fi
  done
done
