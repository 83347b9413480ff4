mkdir -p gpurun_out
timeout 900 python bench.py --config msd > gpurun_out/r2_bench_msd_full.json 2> gpurun_out/r2_bench_msd_full.err
python -c "import json;d=json.load(open('gpurun_out/r2_bench_msd_full.json'));print('msd', d['value'], d['ms_per_step'], d['fit'])"
timeout 900 python bench.py --config higgs --steps 5 > gpurun_out/r2_bench_higgs_full.json 2> gpurun_out/r2_bench_higgs_full.err
python -c "import json;d=json.load(open('gpurun_out/r2_bench_higgs_full.json'));print('higgs', d['value'], d['ms_per_step'], d['fit'])"
timeout 1500 python bench.py --config taxi --steps 2 --warmup 3 --fit-iters 7 > gpurun_out/r2_bench_taxi_fit.json 2> gpurun_out/r2_bench_taxi_fit.err
python -c "import json;d=json.load(open('gpurun_out/r2_bench_taxi_fit.json'));print('taxi', d['value'], d['ms_per_step'], d['fit'])"
