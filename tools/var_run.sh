# A/B runs of variant libraries built with NB_LIBPATH/NB_NVCC_EXTRA (see _build.py); no rebuild on the box
export NB_NO_BUILD=1
for rep in 1 2; do
for v in prev nb; do
  lib=$PWD/paper_2503_02134_b200/libnb_$v.so; [ $v = nb ] && lib=$PWD/paper_2503_02134_b200/libnb.so
  NB_LIBPATH=$lib python tools/sweep.py --cases 16x16x16p7 32x32x32p7 32x32x32p9d --policies fp64 fp32 mixed --iters 200 --reps 3 > gpurun_out/var_${v}_$rep.log 2>&1
done
done
