#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2006_10350_b200.build > gpurun_out/gsc1_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_gsc.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gsc1_pytest_gsc.txt 2>&1
echo "exit $?" >> gpurun_out/gsc1_pytest_gsc.txt
timeout 600 python scripts/precond_probe.py > gpurun_out/gsc1_probe.json 2> gpurun_out/gsc1_probe.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider --deselect tests/test_gpu_gsc.py > gpurun_out/gsc1_pytest_all.txt 2>&1
echo "exit $?" >> gpurun_out/gsc1_pytest_all.txt
