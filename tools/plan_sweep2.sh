#!/bin/bash
# tools/plan_sweep2.sh "cfg:layer:v,s cfg:layer:v,s ..."
for item in $@; do
  IFS=: read c l vs <<< "$item"
  echo -n "$l [$vs]: "; SMMC_FORCE_PLAN=$vs python tools/prof_layer.py --config $c --layer $l --iters 20 2>&1 | tail -1
done
