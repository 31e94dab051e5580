#!/bin/bash
# A/B of stem-kernel thread tiles: tools/stem_variants.py builds lib/ab/*.so;
# "tiled" = SMMC_STEM=0 (the implicit-GEMM kernel), "main" = the in-tree library.
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
for rep in 1 2; do
 for v in main a6 a7 a8; do
  e=""; [ $v != main ] && e="SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so"
  run $v "$e" 3 conv11x11s4_3to96@227_n8
 done
 run tiled SMMC_STEM=0 3 conv7x7s2p3_3to64@224_n8
 for v in main b1 b2 b3; do
  e=""; [ $v != main ] && e="SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so"
  run $v "$e" 3 conv7x7s2p3_3to64@224_n8
 done
 run tiled SMMC_STEM=0 4 vgg01_3to64@224_n64
 for v in c1 c2 c3; do
  run $v "SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so" 4 vgg01_3to64@224_n64
 done
done
