#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/precond_probe.py > gpurun_out/probe1.json 2> gpurun_out/probe1.err
PROBE_M=12000 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/probe1_precond_launches.csv python scripts/precond_probe.py > gpurun_out/probe1_ncu.log 2>&1
