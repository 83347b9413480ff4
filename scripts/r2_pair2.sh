mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_product.py tests/test_gpu_accum64.py tests/test_gpu_cluster.py tests/test_gpu_single_eval.py -x -q > gpurun_out/r2_pair2_pytest.txt 2>&1; tail -3 gpurun_out/r2_pair2_pytest.txt
for c in msd higgs; do for p in 1 0; do
FALKON_TC_PAIR=$p timeout 600 python bench.py --config $c --steps 5 --warmup 3 --quick > gpurun_out/r2_pair2_${c}_$p.json 2> gpurun_out/r2_pair2_${c}_$p.err
python -c "import json;d=json.load(open('gpurun_out/r2_pair2_${c}_$p.json'));print('$c pair=$p', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['roofline']['frac_product'],3))"
done; done
for p in 1 0; do
FALKON_TC_PAIR=$p timeout 600 python bench.py --config taxi --n 50000000 --steps 3 --warmup 3 --quick > gpurun_out/r2_pair2_taxi_$p.json 2> gpurun_out/r2_pair2_taxi_$p.err
python -c "import json;d=json.load(open('gpurun_out/r2_pair2_taxi_$p.json'));print('taxi5e7 pair=$p', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['roofline']['frac_product'],3))"
done
