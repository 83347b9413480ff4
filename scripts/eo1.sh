#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for e in 0 2 3 1; do
  timeout 300 python bench.py --quick --steps 10 --exp-offload $e > gpurun_out/eo1_msd_$e.json 2> gpurun_out/eo1_msd_$e.err
done
timeout 300 python -m pytest tests/test_gpu_product.py -q -k "tensor" --timeout 120 -p no:cacheprovider > gpurun_out/eo1_pytest.txt 2>&1
