#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 300 -p no:cacheprovider > gpurun_out/mo1_pytest_multi.txt 2>&1
echo "exit $?" >> gpurun_out/mo1_pytest_multi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider --deselect tests/test_gpu_multi.py > gpurun_out/mo1_pytest_all.txt 2>&1
echo "exit $?" >> gpurun_out/mo1_pytest_all.txt
