#!/bin/bash
# Background queue of oracle golden fits (CPU only; see scripts/oracle_golden.py).
# One at a time: each holds two m x m fp64 buffers (40 GB at m = 5e4).
cd "$(dirname "$0")/.."
run() { python scripts/oracle_golden.py "$@" --workers 7 >> profiles/r2_oracle_golden.jsonl 2>> /tmp/oracle_queue.err; }
run --config higgs --n 1050000 --m 50000 --direct-max-d 16
run --config taxi --n 2000000 --m 50000
run --config timit --m 50000
