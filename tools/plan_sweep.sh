#!/bin/bash
# Sweep forced (tile variant, split) plans for one layer: tools/plan_sweep.sh CONFIG LAYER "v,s v,s ..."
cfg=$1; layer=$2; shift 2
for vs in $@; do
  echo -n "$vs: "; SMMC_FORCE_PLAN=$vs python tools/prof_layer.py --config $cfg --layer $layer --iters 50 2>&1 | tail -1
done
