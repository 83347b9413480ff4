#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_multi.py -q --timeout 300 -p no:cacheprovider > gpurun_out/mo2_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/mo2_pytest.txt
timeout 600 python scripts/trsv_probe.py > gpurun_out/mo2_trsv.json 2> gpurun_out/mo2_trsv.err
PROBE_LIB=0 PROBE_WARPS=2 PROBE_OUTER=8 PROBE_M=20000 timeout 600 ncu --set full --clock-control none -k regex:"gemm_f64" -s 40 -c 12 -o gpurun_out/mo2_gemm python scripts/precond_probe.py > gpurun_out/mo2_ncu.log 2>&1
timeout 1500 python scripts/fit_parity.py --config higgs --n 1050000 --m 4000 > gpurun_out/mo2_fitpar_higgs.json 2>&1
