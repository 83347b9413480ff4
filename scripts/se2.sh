#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --config timit --quick --steps 3 --single-eval 1 > gpurun_out/se2_timit_1.json 2> gpurun_out/se2_timit_1.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tc_kvp_kernel -c 4 --csv python bench.py --config timit --quick --steps 1 --warmup 1 --single-eval 1 --n 200000 > gpurun_out/se2_ncu.csv 2> gpurun_out/se2_ncu.err
