for v in vA vB vC vD vE vF vG; do NB_MEGA_TMA=0 NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_$v.so python tools/sweep.py --cases 16x16x16p7 32x32x32p7 --iters 100 --reps 2 > gpurun_out/var_$v.log 2>&1; done
NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_vE.so python tools/sweep.py --cases 16x16x16p7 32x32x32p7 --iters 100 --reps 2 > gpurun_out/var_tma.log 2>&1
