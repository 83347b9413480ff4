#!/bin/bash
# GPU gate: full pytest -m gpu + smoke (+ optional extra command in $EXTRA); outputs in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-gate}
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
