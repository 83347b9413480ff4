#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gsc.py tests/test_gpu_fit.py -q --timeout 300 -p no:cacheprovider > gpurun_out/gsc3_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/gsc3_pytest.txt
PROBE_OUTER=2,4,8 PROBE_M=20000,50000 timeout 900 python scripts/precond_probe.py > gpurun_out/gsc3_probe.json 2> gpurun_out/gsc3_probe.err
