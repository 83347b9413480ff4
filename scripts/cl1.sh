#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cluster.py -q --timeout 120 -p no:cacheprovider -x > gpurun_out/cl1_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/cl1_pytest.txt
for c in 1 2; do
  timeout 300 python bench.py --quick --steps 10 --tc-cluster $c > gpurun_out/cl1_msd_$c.json 2> gpurun_out/cl1_msd_$c.err
  timeout 600 python bench.py --config timit --quick --steps 3 --tc-cluster $c --single-eval 0 > gpurun_out/cl1_timit_tp_$c.json 2> gpurun_out/cl1_timit_tp_$c.err
  timeout 600 python bench.py --config timit --quick --steps 3 --tc-cluster $c --single-eval 1 > gpurun_out/cl1_timit_se_$c.json 2> gpurun_out/cl1_timit_se_$c.err
done
