# A/B runs of variant libraries built with NB_LIBPATH/NB_NVCC_EXTRA (see _build.py); no rebuild on the box
export NB_NO_BUILD=1
for v in V1 V2 V3 V4 V5; do NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_$v.so python tools/sweep.py --cases 16x16x16p7 32x32x32p7 --policies mixed fp32 --iters 100 --reps 2 > gpurun_out/var_$v.log 2>&1; done
