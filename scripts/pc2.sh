#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PROBE_LIB=0 PROBE_WARPS=8,2 PROBE_OUTER=8 PROBE_M=20000,50000 timeout 900 python scripts/precond_probe.py > gpurun_out/pc2_probe.json 2> gpurun_out/pc2_probe.err
PROBE_LIB=0 PROBE_WARPS=2 PROBE_OUTER=8 PROBE_M=12000 timeout 600 ncu --set full --clock-control none -k regex:"gemm_f64" -s 20 -c 3 -o gpurun_out/pc2_prof python scripts/precond_probe.py > gpurun_out/pc2_ncu.log 2>&1
