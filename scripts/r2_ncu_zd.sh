# ncu --set full of the ACCUM_F64 tensor kernel vs the fp32 one (HIGGS shape, 1.05M rows)
mkdir -p gpurun_out
for a in 1 0; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_kvp_kernel -c 1 \
  -o gpurun_out/r2_ncu_higgs_acc$a -f python bench.py --config higgs --n 1050000 --steps 1 --warmup 1 --quick --accum-f64 $a > gpurun_out/r2_ncu_higgs_acc$a.log 2>&1
tail -2 gpurun_out/r2_ncu_higgs_acc$a.log
done
