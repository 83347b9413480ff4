#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for CFG in higgs taxi; do
  N=""; [ $CFG = taxi ] && N="--n 50000000"
  for EO in 0 2 3; do
    timeout 600 python bench.py --config $CFG $N --path tensor --exp-offload $EO --quick --steps 3 --warmup 1 > gpurun_out/sdtc_${CFG}_eo$EO.json 2> gpurun_out/sdtc_${CFG}_eo$EO.err
  done
done
