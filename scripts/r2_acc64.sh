# ACCUM_F64: GPU parity + cost per config (one gpurun call)
mkdir -p gpurun_out
./scripts/probes/pipe_rates 1965 > gpurun_out/r2_pipe_rates.txt 2>&1; cat gpurun_out/r2_pipe_rates.txt
timeout 900 python -m pytest tests/test_gpu_accum64.py -x -q > gpurun_out/r2_acc64_pytest.txt 2>&1
tail -3 gpurun_out/r2_acc64_pytest.txt
for c in msd higgs; do
 for a in 0 1; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --quick --accum-f64 $a > gpurun_out/r2_acc64_${c}_$a.json 2> gpurun_out/r2_acc64_${c}_$a.err
  python -c "import json;d=json.load(open('gpurun_out/r2_acc64_${c}_$a.json'));print('$c acc=$a', d['value'], d['ms_per_step'])"
 done
done
