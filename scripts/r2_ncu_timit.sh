mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_kvp_kernel --launch-skip 2 -c 1 -o gpurun_out/r2_ncu_timit_kst -f python bench.py --config timit --steps 1 --warmup 1 --quick > gpurun_out/r2_ncu_timit_kst.log 2>&1
tail -1 gpurun_out/r2_ncu_timit_kst.log
