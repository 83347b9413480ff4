#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/gsc_diag.py 4097 257 90 7.0 > gpurun_out/gsc2_diag90.json 2>&1
timeout 600 python scripts/gsc_diag.py 20000 500 28 5.0 > gpurun_out/gsc2_diag28.json 2>&1
