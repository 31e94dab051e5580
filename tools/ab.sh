#!/bin/bash
# A/B two builds in one box session: tools/ab.sh "config:layer ..." lib1.so lib2.so ...
layers=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  for cl in $layers; do
    c=${cl%%:*}; l=${cl#*:}
    echo -n "$(basename $lib) "; SMMC_LIB=$lib python tools/prof_layer.py --config $c --layer $l --iters 20 2>&1 | tail -1
  done
done
done
