mkdir -p gpurun_out
{ nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp; } > gpurun_out/box_info.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_head.txt 2>&1
tail -3 gpurun_out/r2_pytest_head.txt
