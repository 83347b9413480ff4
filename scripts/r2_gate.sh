# round-2 gate: GPU suite, smoke, default bench line, ACCUM_F64 cost
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.txt 2>&1
tail -3 gpurun_out/r2_pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -2 gpurun_out/r2_smoke.txt
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; tail -c 600 gpurun_out/r2_bench_default.json
for c in msd higgs; do
 for a in 0 1; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --quick --accum-f64 $a > gpurun_out/r2_acc64_${c}_$a.json 2> gpurun_out/r2_acc64_${c}_$a.err
  python -c "import json;d=json.load(open('gpurun_out/r2_acc64_${c}_$a.json'));print('$c acc=$a', d['value'], d['ms_per_step'])"
 done
done
