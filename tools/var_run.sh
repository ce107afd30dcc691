# A/B runs of variant libraries built with NB_LIBPATH/NB_NVCC_EXTRA (see _build.py); no rebuild on the box
export NB_NO_BUILD=1
NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_pa1.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/var_tests.log 2>&1
for rep in 1 2; do
for v in pa0 pa1; do NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_$v.so python tools/sweep.py --cases 16x16x16p7 24x24x24p9 20x20x20p11 --policies mixed fp64 --iters 200 --reps 3 > gpurun_out/var_${v}_$rep.log 2>&1; done
done
