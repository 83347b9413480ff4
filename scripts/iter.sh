#!/bin/bash
# quick iteration: product parity tests + bench (product only) + optional ncu of the tc kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 600 python -m pytest tests/test_gpu_product.py -q --timeout 200 -p no:cacheprovider -x > gpurun_out/pytest_${TAG}.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.txt
timeout 600 python bench.py --quick ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tc_kvp} -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-2} \
  -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 1 --quick ${BENCH_ARGS:-} > gpurun_out/ncu_${TAG}.log 2>&1
fi
