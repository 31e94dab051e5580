run() { echo -n "$1 "; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1; }
L=paper_2411_15659_b200/lib/ab
for rep in 1 2; do
 run main "" 3 conv11x11s4_3to96@227_n8
 for v in a9 a10; do run $v SMMC_LIB=$L/$v.so 3 conv11x11s4_3to96@227_n8; done
 run main "" 3 conv7x7s2p3_3to64@224_n8
 for v in b1 b4 b5 b6; do run $v SMMC_LIB=$L/$v.so 3 conv7x7s2p3_3to64@224_n8; done
 run tiled SMMC_STEM=0 4 vgg01_3to64@224_n64
 for v in c1 c2 c4; do run $v SMMC_LIB=$L/$v.so 4 vgg01_3to64@224_n64; done
done
