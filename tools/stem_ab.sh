#!/bin/bash
L="3:conv7x7s2p3_3to64@224_n8 3:conv11x11s4_3to96@227_n8 4:vgg01_3to64@224_n64"
for rep in 1 2; do
 for v in tiled main; do
  for cl in $L; do c=${cl%%:*}; l=${cl#*:}
   case $v in
    tiled) e="SMMC_STEM=0";; main) e="";; *) e="SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so";;
   esac
   echo -n "$v "; env $e python tools/prof_layer.py --config $c --layer $l --iters 20 2>&1 | tail -1
  done
 done
done
