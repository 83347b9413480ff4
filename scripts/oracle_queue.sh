#!/bin/bash
# Background queue of oracle golden fits (CPU only; see scripts/oracle_golden.py).
cd "$(dirname "$0")/.."
while pgrep -f "oracle_golden.py --config taxi --n 2000000" > /dev/null; do sleep 30; done
run() { python scripts/oracle_golden.py "$@" --workers 7 >> profiles/r2_oracle_golden.jsonl 2>> /tmp/oracle_queue.err; }
run --config higgs --n 1050000 --m 50000 --direct-max-d 16
run --config timit --m 50000
