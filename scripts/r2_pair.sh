mkdir -p gpurun_out
FALKON_TC_PAIR=1 timeout 300 python scripts/pair_check.py > gpurun_out/r2_pair_check.txt 2>&1; cat gpurun_out/r2_pair_check.txt | tail -8
for p in 1 0; do
FALKON_TC_PAIR=$p timeout 600 python bench.py --config timit --steps 5 --warmup 3 --quick > gpurun_out/r2_pair_timit_$p.json 2> gpurun_out/r2_pair_timit_$p.err
python -c "import json;d=json.load(open('gpurun_out/r2_pair_timit_$p.json'));print('pair=$p', d['value'], d['ms_per_step'], d['kernel_ms']['pass_a'], d['kernel_ms']['pass_b'], d['clocks']['sm_mhz'], d['roofline']['frac'])"
FALKON_TC_PAIR=$p timeout 600 python bench.py --config timit --single-eval 0 --steps 3 --warmup 2 --quick > gpurun_out/r2_pair_timit2p_$p.json 2> gpurun_out/r2_pair_timit2p_$p.err
python -c "import json;d=json.load(open('gpurun_out/r2_pair_timit2p_$p.json'));print('two-pass pair=$p', d['value'], d['ms_per_step'], d['kernel_ms']['pass_a'], d['clocks']['sm_mhz'], d['roofline']['frac'])"
done
