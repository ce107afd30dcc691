# A/B of standalone ops across library variants: bash tools/ab_ops.sh <prefix> "<cases>" "<policies>" v1 v2 ...
pre=$1; cases=$2; pols=$3; shift 3
mkdir -p gpurun_out/r2
export NB_NO_BUILD=1
for v in "$@"; do
  lib=$PWD/paper_2503_02134_b200/libnb_$v.so; [ $v = nb ] && lib=$PWD/paper_2503_02134_b200/libnb.so
  NB_LIBPATH=$lib timeout 600 python tools/bench_ops.py --cases $cases --policies $pols > gpurun_out/r2/${pre}_$v.log 2>&1
  NB_DSSUM=csr NB_LIBPATH=$lib timeout 600 python tools/bench_ops.py --cases $cases --policies $pols > gpurun_out/r2/${pre}_${v}_csr.log 2>&1
done
