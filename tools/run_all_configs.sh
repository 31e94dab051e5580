#!/bin/bash
# Bench every BASELINE config (1-GPU), per-layer details into gpurun_out/.
set -u
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --cpu-seconds ${CPU_S:-5} \
     --details gpurun_out/bench_cfg$c.json > gpurun_out/bench_cfg$c.log 2>&1
  echo "config $c rc=$?"
done
