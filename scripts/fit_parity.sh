#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/fitpar_host.txt; free -g >> gpurun_out/fitpar_host.txt
timeout 900 python scripts/fit_parity.py --config msd --m 5000 > gpurun_out/fitpar_msd.json 2>&1
timeout 900 python scripts/fit_parity.py --config timit --m 4000 > gpurun_out/fitpar_timit.json 2>&1
timeout 900 python scripts/fit_parity.py --config higgs --n 1050000 --m 8000 > gpurun_out/fitpar_higgs.json 2>&1
timeout 900 python scripts/fit_parity.py --config taxi --n 2000000 --m 5000 > gpurun_out/fitpar_taxi.json 2>&1
timeout 600 python scripts/fit_parity.py --config msd --n 200000 --m 3000 --kernel 1 > gpurun_out/fitpar_msd_lap.json 2>&1
