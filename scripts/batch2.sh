#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_product.py tests/test_gpu_fit.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_b2.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_b2.txt
for CFG in higgs taxi; do
  N=""; [ $CFG = taxi ] && N="--n 50000000"
  timeout 600 python bench.py --config $CFG $N --path simt --quick --steps 3 --warmup 1 > gpurun_out/b2_simt_$CFG.json 2>&1
  FALKON_TC_EPIW=16 timeout 600 python bench.py --config $CFG $N --quick --steps 3 --warmup 1 > gpurun_out/b2_epi16_$CFG.json 2>&1
  FALKON_TC_EPIW=16 timeout 600 python bench.py --config $CFG $N --exp-offload 2 --quick --steps 3 --warmup 1 > gpurun_out/b2_epi16eo2_$CFG.json 2>&1
done
FALKON_TC_EPIW=16 timeout 600 python bench.py --quick --steps 5 --warmup 2 > gpurun_out/b2_epi16_msd.json 2>&1
timeout 600 python scripts/fit_profile.py > gpurun_out/b2_fit_msd.json 2>&1
