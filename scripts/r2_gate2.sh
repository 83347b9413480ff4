mkdir -p gpurun_out
PYTHONPATH=scripts timeout 900 python scripts/crossover.py > gpurun_out/r2_crossover.jsonl 2>&1; tail -2 gpurun_out/r2_crossover.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_timit.csv python bench.py --steps 2 --warmup 3 --quick > gpurun_out/r2_launches_timit.log 2>&1; tail -1 gpurun_out/r2_launches_timit.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu2.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu2.txt
