mkdir -p gpurun_out
for f in 0 1; do
FALKON_FUSED_GEMV=$f timeout 600 python bench.py --config timit --steps 5 --warmup 3 --quick > gpurun_out/r2_se2_timit_f$f.json 2> gpurun_out/r2_se2_timit_f$f.err
python -c "import json;d=json.load(open('gpurun_out/r2_se2_timit_f$f.json'));print('fused=$f', d['value'], d['ms_per_step'], d['kernel_ms']['pass_a'], d['kernel_ms']['pass_b'], d['clocks']['sm_mhz'])"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_kvp_kernel --launch-skip 3 -c 1 -o gpurun_out/r2_ncu_timit_fused -f python bench.py --config timit --n 200000 --steps 1 --warmup 1 --quick > gpurun_out/r2_ncu_timit_fused.log 2>&1
tail -1 gpurun_out/r2_ncu_timit_fused.log
