#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_gsc.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/tr1_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/tr1_pytest.txt
timeout 600 python scripts/trsv_probe.py > gpurun_out/tr1_trsv.json 2> gpurun_out/tr1_trsv.err
timeout 900 python bench.py > gpurun_out/tr1_bench.json 2> gpurun_out/tr1_bench.err
