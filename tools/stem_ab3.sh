#!/bin/bash
# A/B of 11x11 s4 stem-kernel thread tiles (lib/ab/v*.so built with STEM_V3 + SV_* defines)
for rep in 1 2; do
 for v in main v1 v2 v3 v4 v5; do
  e=""; [ $v != main ] && e="SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so"
  echo -n "$v "; env $e python tools/prof_layer.py --config 3 --layer conv11x11s4_3to96@227_n8 --iters 20 2>&1 | tail -1
 done
done
