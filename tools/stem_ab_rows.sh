#!/bin/bash
# A/B of multi-row (R = 2) stem thread tiles (lib/ab/r*.so, tools/stem_variants.py)
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
L=paper_2411_15659_b200/lib/ab
for v in r1a r1b r2a r2b r2c r2d r3a r3b r3c; do  # needs tools/experiments/stem_multirow.patch applied
  echo -n "parity $v: "; SMMC_LIB=$L/$v.so timeout 300 python -m pytest tests/test_gpu_stem.py -q -x 2>&1 | tail -1
done
for rep in 1; do
 run main "" 3 conv7x7s2p3_3to64@224_n8
 for v in r2a r2b r2c r2d; do run $v SMMC_LIB=$L/$v.so 3 conv7x7s2p3_3to64@224_n8; done
 run main "" 3 conv11x11s4_3to96@227_n8
 for v in r3a r3b r3c; do run $v SMMC_LIB=$L/$v.so 3 conv11x11s4_3to96@227_n8; done
 run main "" 4 vgg01_3to64@224_n64
 for v in r1a r1b; do run $v SMMC_LIB=$L/$v.so 4 vgg01_3to64@224_n64; done
done
