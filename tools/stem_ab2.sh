cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_ab2.log; : > $O
run() { echo -n "$1 $3 " >> $O; env $2 python tools/prof_layer.py --config 3 --layer $3 --iters 20 2>&1 | tail -1 >> $O; }
for v in paper_2411_15659_b200/lib/ab/m*.so; do
  echo -n "tests $v: " >> $O
  SMMC_LIB=$v python -m pytest tests/test_gpu_stem.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $O
done
for rep in 1 2; do
  run main "" conv7x7s2p3_3to64@224_n8
  for v in paper_2411_15659_b200/lib/ab/m2*.so; do run $(basename $v .so) SMMC_LIB=$v conv7x7s2p3_3to64@224_n8; done
  run main "" conv11x11s4_3to96@227_n8
  for v in paper_2411_15659_b200/lib/ab/m3*.so; do run $(basename $v .so) SMMC_LIB=$v conv11x11s4_3to96@227_n8; done
done
cat $O
