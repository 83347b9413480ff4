#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for M in 0 8 9 10; do
  FALKON_TC_MODE=$M timeout 600 python bench.py --config higgs --n 3000000 --quick --steps 3 --warmup 1 > gpurun_out/dsm_m$M.json 2> gpurun_out/dsm_m$M.err
done
