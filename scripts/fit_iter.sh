#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-fi}
timeout 900 python -m pytest tests/test_gpu_fit.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fit_${TAG}.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_fit_${TAG}.txt
timeout 600 python scripts/fit_profile.py --repeat 1 > gpurun_out/fitprof_msd_${TAG}.json 2>&1
