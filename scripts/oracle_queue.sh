#!/bin/bash
# Background queue of oracle golden fits (CPU only; see scripts/oracle_golden.py).
cd "$(dirname "$0")/.."
run() { python scripts/oracle_golden.py "$@" --workers 7 >> profiles/r2_oracle_golden.jsonl 2>> /tmp/oracle_queue.err; }
run --config msd
run --config taxi --n 2000000 --m 50000
run --config timit --m 50000
run --config higgs --n 1050000 --m 50000
