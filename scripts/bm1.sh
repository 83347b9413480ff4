#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --multi-k 16 > gpurun_out/bm1_msd.json 2> gpurun_out/bm1_msd.err
timeout 900 python bench.py --config timit --no-fit --steps 5 --multi-k 144 --oracle-seconds 8 > gpurun_out/bm1_timit.json 2> gpurun_out/bm1_timit.err
timeout 1500 python bench.py --config higgs --steps 5 --gsc-config higgs_log --oracle-seconds 8 > gpurun_out/bm1_higgs.json 2> gpurun_out/bm1_higgs.err
