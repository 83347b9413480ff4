#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for M in ${MODES:-0 1 2 3 8 9}; do
  FALKON_TC_MODE=$M timeout 300 python bench.py --quick --steps 5 --warmup 2 > gpurun_out/sweep_mode$M.json 2>gpurun_out/sweep_mode$M.err
done
for M in ${TMODES:-1 2 3}; do
  FALKON_TC_MODE=$M timeout 300 python -m pytest tests/test_gpu_product.py -q -k tensor --timeout 200 -p no:cacheprovider > gpurun_out/sweep_pytest_mode$M.txt 2>&1
done
