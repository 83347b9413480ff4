#!/bin/bash
# full GPU gate: pytest -m gpu, smoke, default bench; outputs in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-full}
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench exit $?" >> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
