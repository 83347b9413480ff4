#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_gsc.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pc1_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/pc1_pytest.txt
PROBE_LIB=0 PROBE_WARPS=8,16 PROBE_OUTER=4,8 PROBE_M=20000,50000 timeout 900 python scripts/precond_probe.py > gpurun_out/pc1_probe.json 2> gpurun_out/pc1_probe.err
PROBE_LIB=0 PROBE_WARPS=16 PROBE_OUTER=8 PROBE_M=12000 timeout 600 ncu --set full --clock-control none -k regex:"gemm_f64|potrf_diag" -s 20 -c 6 -o gpurun_out/pc1_prof python scripts/precond_probe.py > gpurun_out/pc1_ncu.log 2>&1
