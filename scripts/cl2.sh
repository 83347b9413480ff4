#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 1 2; do
  timeout 300 python bench.py --config higgs --n 2100000 --quick --steps 5 --tc-cluster $c > gpurun_out/cl2_higgs_$c.json 2> gpurun_out/cl2_higgs_$c.err
  timeout 300 python bench.py --config taxi --n 20000000 --quick --steps 3 --tc-cluster $c > gpurun_out/cl2_taxi_$c.json 2> gpurun_out/cl2_taxi_$c.err
done
for e in 2 3; do
  timeout 300 python bench.py --config higgs --n 2100000 --quick --steps 5 --tc-cluster 1 --exp-offload $e > gpurun_out/cl2_higgs_e$e.json 2> gpurun_out/cl2_higgs_e$e.err
  timeout 300 python bench.py --config taxi --n 20000000 --quick --steps 3 --tc-cluster 1 --exp-offload $e > gpurun_out/cl2_taxi_e$e.json 2> gpurun_out/cl2_taxi_e$e.err
done
