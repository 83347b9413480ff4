#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_product.py -q -k "offload" --timeout 120 -p no:cacheprovider > gpurun_out/eo2_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/eo2_pytest.txt
for e in 0 4 5 0; do
  timeout 300 python bench.py --config higgs --n 2100000 --quick --steps 5 --exp-offload $e > gpurun_out/eo2_higgs_$e.json 2> gpurun_out/eo2_higgs_$e.err
  timeout 300 python bench.py --config taxi --n 20000000 --quick --steps 3 --exp-offload $e > gpurun_out/eo2_taxi_$e.json 2> gpurun_out/eo2_taxi_$e.err
done
