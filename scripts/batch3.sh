#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python scripts/fit_parity.py --config higgs --n 1050000 --m 8000 > gpurun_out/fitpar3_higgs.json 2>&1
timeout 900 python scripts/fit_parity.py --config taxi --n 2000000 --m 5000 > gpurun_out/fitpar3_taxi.json 2>&1
timeout 600 python scripts/fit_parity.py --config msd --n 50000 --m 2000 --kernel 1 > gpurun_out/fitpar3_msd_lap.json 2>&1
timeout 900 python bench.py --config taxi --steps 2 --warmup 1 --oracle-seconds 10 > gpurun_out/bench_taxi_full.json 2> gpurun_out/bench_taxi_full.err
