cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_ab2.log; : > $O
run() { echo -n "$1 $3 " >> $O; env $2 python tools/prof_layer.py --config 3 --layer $3 --iters 20 2>&1 | tail -1 >> $O; }
for rep in 1 2; do
  run main "" conv7x7s2p3_3to64@224_n8
  for v in m2a m2b m2c m2d m2e; do run $v SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so conv7x7s2p3_3to64@224_n8; done
  run main "" conv11x11s4_3to96@227_n8
  for v in; do run $v SMMC_LIB=paper_2411_15659_b200/lib/ab/$v.so conv11x11s4_3to96@227_n8; done
done
cat $O
