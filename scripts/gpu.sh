#!/bin/bash
# One parameterised driver for the GPU-box runs behind profiles/ (replaces the one-off wrappers).
#   gpurun --timeout 1800 -- 'bash scripts/gpu.sh TASK [ARGS]'      outputs in gpurun_out/
# TASK:
#   gate [TAG]                 pytest -m gpu + smoke
#   bench CFG [TAG] [ARGS..]   one bench.py line (ARGS passed through, e.g. --quick --steps 5)
#   ab CFG "ENV=V .." ..       bench --quick once per environment setting (A/B of a variant)
#   launches CFG [TAG]         ncu launch list (per-launch gpu__time_duration) + summary
#   ncu CFG KREGEX [TAG] [SKIP] one `ncu --set full` capture of the first matching launch
#   traffic CFG KREGEX [TAG]   dram / lts bytes and time of matching launches
#   fits                       bench lines with the full fit on MSD, HIGGS, TAXI
#   sweeps                     SIMT/tensor crossover, Fig. mvm_impl n- and d-sweeps
#   sanitize                   compute-sanitizer memcheck / racecheck / synccheck
#   reference [CFG]            the oracle arm (bench.py --impl reference)
#   probes                     L2 / HBM bandwidth and pipe-rate microbenchmarks
#   evidence                   round-end bench lines (TIMIT headline + launch list, MSD, HIGGS, TAXI)
#   ozaki [M ...]              preconditioner builds, Ozaki vs DMMA GEMMs (scripts/ozaki_probe.py)
#   configscale                the -m gpu slow config-scale fit parity against tests/golden/fits
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
task=$1; shift
case $task in
gate)
  TAG=${1:-gate}
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt; tail -3 gpurun_out/pytest_gpu_$TAG.txt
  timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.txt 2>&1
  echo "smoke exit $?" >> gpurun_out/smoke_$TAG.txt; tail -2 gpurun_out/smoke_$TAG.txt ;;
bench)
  CFG=$1; TAG=${2:-b}; shift 2
  timeout 1800 python bench.py --config $CFG "$@" > gpurun_out/bench_${CFG}_$TAG.json 2> gpurun_out/bench_${CFG}_$TAG.err
  echo "bench exit $?"; tail -c 1500 gpurun_out/bench_${CFG}_$TAG.json ;;
ab)
  CFG=$1; shift
  for e in "$@"; do
    t=$(echo "$e" | tr ' =' '_-')
    env $e timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 --quick > gpurun_out/ab_${CFG}_$t.json 2> gpurun_out/ab_${CFG}_$t.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${CFG}_$t.json'));print('$e', round(d['ms_per_step'],2), {k:round(v,1) for k,v in d['kernel_ms'].items() if v}, d['clocks']['sm_mhz'], d['roofline'].get('frac'), d['roofline'].get('frac_product'))" || tail -3 gpurun_out/ab_${CFG}_$t.err
  done ;;
launches)
  CFG=$1; TAG=${2:-l}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${CFG}_$TAG.csv python bench.py --config $CFG --steps 2 --warmup 3 --quick \
    > gpurun_out/launches_${CFG}_$TAG.log 2>&1
  python scripts/launch_list.py gpurun_out/launches_${CFG}_$TAG.csv | tee gpurun_out/launches_${CFG}_$TAG.txt ;;
ncu)
  CFG=$1; K=$2; TAG=${3:-n}; SKIP=${4:-2}
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip $SKIP -c 1 \
    -o gpurun_out/ncu_${CFG}_$TAG -f python bench.py --config $CFG --steps 1 --warmup 1 --quick \
    > gpurun_out/ncu_${CFG}_$TAG.log 2>&1
  echo "ncu exit $?"; python scripts/ncu_summary.py gpurun_out/ncu_${CFG}_$TAG.ncu-rep | tee gpurun_out/ncu_${CFG}_$TAG.txt ;;
traffic)
  CFG=$1; K=$2; TAG=${3:-t}
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    -k regex:$K --launch-skip 6 -c 2 --csv python bench.py --config $CFG --steps 2 --warmup 3 --quick \
    > gpurun_out/traffic_${CFG}_$TAG.csv 2>&1
  grep -E "dram__bytes|gpu__time|lts__t_bytes" gpurun_out/traffic_${CFG}_$TAG.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' ;;
fits)
  for c in msd higgs; do bash "$0" bench $c fit --steps 5; done
  bash "$0" bench taxi fit --steps 2 --warmup 3 ;;
sweeps)
  PYTHONPATH=scripts timeout 900 python scripts/crossover.py > gpurun_out/crossover.jsonl 2>&1; tail -2 gpurun_out/crossover.jsonl
  timeout 1500 python scripts/mvm_sweep.py all > gpurun_out/mvm_sweep.jsonl 2>&1; tail -2 gpurun_out/mvm_sweep.jsonl ;;
sanitize)
  for t in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitize_$t.txt 2>&1
    echo "$t rc=$?"; tail -3 gpurun_out/sanitize_$t.txt
  done ;;
reference)
  timeout 900 python bench.py --impl reference --config ${1:-timit} --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  tail -c 800 gpurun_out/bench_ref.json ;;
probes)
  for p in l2_bw pipe_rates; do
    nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/$p scripts/probes/$p.cu && /tmp/$p | tee gpurun_out/probe_$p.txt
  done ;;
evidence)  # round-end evidence: headline bench, launch list, per-config lines with fits, oracle arm
  bash "$0" bench timit final > /dev/null; tail -c 400 gpurun_out/bench_timit_final.json; echo
  bash "$0" launches timit final | tail -8
  bash "$0" bench msd final > /dev/null
  bash "$0" bench higgs final --steps 5 > /dev/null
  bash "$0" bench taxi final --n 100000000 --steps 3 --fit-iters 7 > /dev/null
  bash "$0" reference timit ;;
ozaki)  # preconditioner build times and per-kernel device time, Ozaki vs DMMA GEMMs
  OZ_KERNELS=1 timeout 900 python scripts/ozaki_probe.py ${1:-20000} ${2:-50000} | tee gpurun_out/ozaki_probe.jsonl ;;
configscale)
  timeout 3000 python -m pytest tests/test_gpu_fit_configscale.py -m gpu -q -rA > gpurun_out/configscale.txt 2>&1
  tail -15 gpurun_out/configscale.txt ;;
*) sed -n 2,17p "$0"; exit 2 ;;
esac
