#!/bin/bash
# Round-end evidence at HEAD: GPU suite + smoke, default bench (MSD) + launch list + ncu full of
# the dominant kernel, TIMIT / HIGGS bench lines, HIGGS pass-A ncu; outputs in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=fin bash scripts/gpu_gate.sh
CFG=msd TAG=fin bash scripts/profile.sh
timeout 900 python bench.py --config timit --steps 3 > gpurun_out/bench_timit_fin.json 2> gpurun_out/bench_timit_fin.err
timeout 900 python bench.py --config higgs --steps 3 > gpurun_out/bench_higgs_fin.json 2> gpurun_out/bench_higgs_fin.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_kvp -s 2 -c 1 \
  -o gpurun_out/prof_higgs_fin python bench.py --config higgs --n 2100000 --steps 1 --warmup 1 --quick \
  > gpurun_out/ncu_full_higgs_fin.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_fin.json 2> gpurun_out/bench_ref_fin.err
