#!/bin/bash
# A/B of the persistent 1x1 block-stream kernel against tiled split-K plans
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
for rep in 1 2; do
 L=conv1x1_256to64@56_n8
 run main "" 3 $L
 run tiled SMMC_1X1=0 3 $L
 for fp in 1,2 1,3 1,4 1,0 3,3 0,3; do run f$fp SMMC_FORCE_PLAN=$fp 3 $L; done
 L=conv1x1_64to256@56_n256
 run main "" 5 $L
 run tiled SMMC_1X1=0 5 $L
 for fp in 3,1 1,1 0,1; do run f$fp SMMC_FORCE_PLAN=$fp 5 $L; done
done
