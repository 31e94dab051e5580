#!/bin/bash
# A/B of stem-kernel occupancy variants (lib/ab/m*.so from tools/stem_variants.py)
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
L=paper_2411_15659_b200/lib/ab
for v in m1a m1b m2a m2b m3a m3b; do
  echo -n "parity $v: "; SMMC_LIB=$L/$v.so timeout 300 python -m pytest tests/test_gpu_stem.py -q -x 2>&1 | tail -1
done
for rep in 1 2; do
 run main "" 3 conv7x7s2p3_3to64@224_n8
 for v in m2a m2b; do run $v SMMC_LIB=$L/$v.so 3 conv7x7s2p3_3to64@224_n8; done
 run main "" 3 conv11x11s4_3to96@227_n8
 for v in m3a m3b; do run $v SMMC_LIB=$L/$v.so 3 conv11x11s4_3to96@227_n8; done
 run main "" 4 vgg01_3to64@224_n64
 for v in m1a m1b; do run $v SMMC_LIB=$L/$v.so 4 vgg01_3to64@224_n64; done
done
