#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_product.py -q -k "tensor or 90" --timeout 200 -p no:cacheprovider > gpurun_out/sw2_pytest_ts.txt 2>&1
FALKON_TC_TS=0 timeout 300 python -m pytest tests/test_gpu_product.py -q -k "tensor or 90" --timeout 200 -p no:cacheprovider > gpurun_out/sw2_pytest_ss.txt 2>&1
for TS in 1 0; do for M in 0 11; do
  FALKON_TC_TS=$TS FALKON_TC_MODE=$M timeout 300 python bench.py --quick --steps 5 --warmup 2 > gpurun_out/sw2_ts${TS}_m$M.json 2>gpurun_out/sw2_ts${TS}_m$M.err
done; done
