mkdir -p gpurun_out/r2
export NB_NO_BUILD=1
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r2/gpu_tests_flat.log
for rep in 1 2; do
for v in prev nb; do
  lib=$PWD/paper_2503_02134_b200/libnb_$v.so; [ $v = nb ] && lib=$PWD/paper_2503_02134_b200/libnb.so
  NB_LIBPATH=$lib python tools/sweep.py --cases 16x16x16p7 32x32x32p7 32x32x32p9d 32x32x32p11 --policies mixed fp32 fp64 --iters 200 --reps 3 > gpurun_out/r2/ab1_${rep}_$v.log 2>&1
done
done
