#!/bin/bash
# bench + ncu launch list + one full ncu capture of the top kernels; outputs in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFG=${CFG:-msd}
TAG=${TAG:-r1}
timeout 900 python bench.py --config $CFG ${BENCH_ARGS:-} > gpurun_out/bench_${CFG}_${TAG}.json 2> gpurun_out/bench_${CFG}_${TAG}.err
echo "bench exit $?" >> gpurun_out/bench_${CFG}_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --steps 2 --warmup 1 --quick \
  > gpurun_out/ncu_launch_${CFG}_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-kvp} -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-2} \
  -o gpurun_out/prof_${CFG}_${TAG} python bench.py --config $CFG --steps 1 --warmup 1 --quick \
  > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_${CFG}_${TAG}.log
