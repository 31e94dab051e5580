#!/bin/bash
# A/B of the stem kernel against the tiled kernel ("tiled" = SMMC_STEM=0);
# thread-tile variants: build lib/ab/*.so with tools/stem_variants.py and add
# them to the loop (SMMC_LIB=...).
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
for rep in 1 2; do
 for l in conv7x7s2p3_3to64@224_n8 conv11x11s4_3to96@227_n8; do
  run tiled SMMC_STEM=0 3 $l
  run main "" 3 $l
 done
done
