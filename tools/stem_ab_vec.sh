#!/bin/bash
# A/B of float4 vector windows (default) against scalar window loads (SMMC_STEM_SCALAR=1)
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
echo -n "parity vec: "; timeout 300 python -m pytest tests/test_gpu_stem.py -q -x 2>&1 | tail -1
for rep in 1 2; do
 run vec7_needs_VOFF1_in_case2 "" 3 conv7x7s2p3_3to64@224_n8
 run scalar SMMC_STEM_SCALAR=1 3 conv7x7s2p3_3to64@224_n8
 run vec "" 4 vgg01_3to64@224_n64
 run scalar SMMC_STEM_SCALAR=1 4 vgg01_3to64@224_n64
done
