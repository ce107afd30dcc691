# A/B/C/D runs of variant library builds (NB_LIBPATH), same session, interleaved
export NB_NO_BUILD=1
i=0
for v in ${AB_LIBS:-prev nb}; do :; done
for rep in 1 2; do
for v in ${AB_LIBS:-prev nb}; do
  i=$((i+1))
  lib=$PWD/paper_2503_02134_b200/libnb_$v.so; [ $v = nb ] && lib=$PWD/paper_2503_02134_b200/libnb.so
  NB_LIBPATH=$lib python tools/sweep.py --cases ${AB_CASES:-32x32x32p7 16x16x16p7} --policies ${AB_POL:-fp32 mixed} --iters 200 --reps 5 > gpurun_out/ab_${rep}_$v.log 2>&1
done
done
