# usage: bash tools/ab_run2.sh <prefix> "<cases>" "<policies>" v1 v2 ...   (v = tag of libnb_<tag>.so, nb = libnb.so)
pre=$1; cases=$2; pols=$3; shift 3
mkdir -p gpurun_out/r2
export NB_NO_BUILD=1
for rep in 1 2; do
for v in "$@"; do
  lib=$PWD/paper_2503_02134_b200/libnb_$v.so; [ $v = nb ] && lib=$PWD/paper_2503_02134_b200/libnb.so
  NB_LIBPATH=$lib timeout 600 python tools/sweep.py --cases $cases --policies $pols --iters 200 --reps 3 ${SWEEP_EXTRA:-} > gpurun_out/r2/${pre}_${rep}_$v.log 2>&1
done
done
