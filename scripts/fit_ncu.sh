#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-fn}
timeout 900 python -m pytest tests/test_gpu_fit.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fit_${TAG}.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_fit_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trsv|gemm_f64" -s 300 -c 4 -o gpurun_out/prof_fit_${TAG} python scripts/fit_profile.py --iters 3 > gpurun_out/ncu_fit_${TAG}.log 2>&1
