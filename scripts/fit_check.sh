#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/fit_profile.py --m 20000 --repeat 1 > gpurun_out/fitprof_m20k.json 2>&1
timeout 600 python scripts/fit_profile.py --repeat 1 > gpurun_out/fitprof_msd.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"trsv|gemm_f64|potrf_diag|kmm" -s 40 -c 6 -o gpurun_out/prof_fit python scripts/fit_profile.py --m 20000 --iters 2 > gpurun_out/ncu_fit.log 2>&1
