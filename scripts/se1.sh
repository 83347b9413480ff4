#!/bin/bash
# single-evaluation strip product: parity tests + TIMIT product timing, SE off vs on
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_single_eval.py tests/test_gpu_product.py -q --timeout 300 -p no:cacheprovider -x > gpurun_out/se1_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/se1_pytest.txt
for se in 0 1; do
  timeout 600 python bench.py --config timit --quick --steps 3 --single-eval $se > gpurun_out/se1_timit_$se.json 2> gpurun_out/se1_timit_$se.err
done
timeout 600 python bench.py --quick --steps 5 --single-eval 1 > gpurun_out/se1_msd_1.json 2> gpurun_out/se1_msd_1.err
