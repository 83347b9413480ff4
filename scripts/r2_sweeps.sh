mkdir -p gpurun_out
timeout 1500 python scripts/mvm_sweep.py all > gpurun_out/r2_mvm_sweep.jsonl 2> gpurun_out/r2_mvm_sweep.err; tail -2 gpurun_out/r2_mvm_sweep.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/r2_sanitize_$t.txt 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/r2_sanitize_$t.txt
done
