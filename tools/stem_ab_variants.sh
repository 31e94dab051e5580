#!/bin/bash
# A/B of stem-kernel thread tiles built by tools/stem_variants.py (lib/ab/*.so)
run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
L=paper_2411_15659_b200/lib/ab
for rep in 1 2; do
 run main "" 4 vgg01_3to64@224_n64
 for v in $(ls $L | sed 's/\.so$//'); do run $v SMMC_LIB=$L/$v.so 4 vgg01_3to64@224_n64; done
done
