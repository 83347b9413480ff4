mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_single_eval.py tests/test_gpu_accum64.py tests/test_gpu_gsc.py tests/test_gpu_product.py -x -q > gpurun_out/r2_se_pytest.txt 2>&1
tail -3 gpurun_out/r2_se_pytest.txt
timeout 600 python bench.py --config timit --steps 5 --warmup 3 --quick > gpurun_out/r2_se_timit.json 2> gpurun_out/r2_se_timit.err
python -c "import json;d=json.load(open('gpurun_out/r2_se_timit.json'));print('timit', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['frac_product'], d['kernel_ms'], d['clocks'])"
