mkdir -p gpurun_out
for v in "1 4" "1 3" "1 2" "0 4"; do set -- $v
FALKON_FUSED_GEMV=$1 FALKON_TC_SST=$2 timeout 600 python bench.py --config timit --steps 5 --warmup 3 --quick > gpurun_out/r2_se3_$1_$2.json 2> gpurun_out/r2_se3_$1_$2.err
python -c "import json;d=json.load(open('gpurun_out/r2_se3_$1_$2.json'));print('fused=$1 sst=$2', d['value'], d['ms_per_step'], d['kernel_ms']['pass_a'], d['kernel_ms']['pass_b'], d['clocks']['sm_mhz'])"
done
