# ncu A/B of one megakernel launch (32^3 p7 fp32, 20 iterations) for two library builds
export NB_NO_BUILD=1
for v in prev nb; do
  lib=$PWD/paper_2503_02134_b200/libnb_$v.so; [ $v = nb ] && lib=$PWD/paper_2503_02134_b200/libnb.so
  NB_LIBPATH=$lib python tools/sweep.py --cases 32x32x32p7 --policies fp32 --iters 20 --reps 1 > gpurun_out/abn_plain_$v.log 2>&1 && \
  NB_LIBPATH=$lib ncu --set full --clock-control none -k regex:k_cg_mega -c 1 -o gpurun_out/abn_$v -f python tools/sweep.py --cases 32x32x32p7 --policies fp32 --iters 20 --reps 1 > gpurun_out/abn_ncu_$v.log 2>&1
done
