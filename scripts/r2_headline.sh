mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gsc.py -x -q > gpurun_out/r2_gsc_pytest.txt 2>&1; tail -2 gpurun_out/r2_gsc_pytest.txt
timeout 900 python bench.py > gpurun_out/r2_bench_timit_pair.json 2> gpurun_out/r2_bench_timit_pair.err; tail -c 300 gpurun_out/r2_bench_timit_pair.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_kvp_kernel --launch-skip 2 -c 1 -o gpurun_out/r2_ncu_timit_pair -f python bench.py --steps 1 --warmup 1 --quick > gpurun_out/r2_ncu_timit_pair.log 2>&1; tail -1 gpurun_out/r2_ncu_timit_pair.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_timit_pair.csv python bench.py --steps 2 --warmup 3 --quick > /dev/null 2>&1
