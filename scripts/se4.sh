#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_kvp_kernel -s 2 -c 1 -o gpurun_out/se4_se python bench.py --config timit --quick --steps 1 --warmup 1 --single-eval 1 --n 171520 > gpurun_out/se4_ncu_se.log 2>&1
