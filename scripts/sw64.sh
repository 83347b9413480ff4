#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_single_eval.py tests/test_gpu_product.py tests/test_gpu_multi.py -q --timeout 200 -p no:cacheprovider -x > gpurun_out/sw64_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/sw64_pytest.txt
for se in 0 1; do
  timeout 600 python bench.py --config timit --quick --steps 3 --single-eval $se > gpurun_out/sw64_timit_$se.json 2> gpurun_out/sw64_timit_$se.err
done
