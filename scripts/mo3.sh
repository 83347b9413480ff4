#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_product.py -q --timeout 300 -p no:cacheprovider > gpurun_out/mo3_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/mo3_pytest.txt
timeout 600 python bench.py --quick --steps 3 --multi-k 16 > gpurun_out/mo3_msd.json 2> gpurun_out/mo3_msd.err
timeout 600 python bench.py --quick --steps 3 --multi-k 8 > gpurun_out/mo3_msd8.json 2> gpurun_out/mo3_msd8.err
timeout 900 python bench.py --config timit --quick --steps 2 --multi-k 32 > gpurun_out/mo3_timit.json 2> gpurun_out/mo3_timit.err
timeout 1200 python scripts/gsc_parity.py --n 200000 --m 2000 > gpurun_out/mo3_gscpar.json 2>&1
