cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_lane.log; : > $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3 >> $O
run() { echo -n "$1 " >> $O; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters ${5:-20} 2>&1 | tail -1 >> $O; }
for rep in 1 2; do
 for cl in 4:vgg02_64to64@224_n64:5 4:vgg04_128to128@112_n64:5 4:vgg06_256to256@56_n64:5 4:vgg09_512to512@28_n64:5 4:vgg12_512to512@14_n64:5 \
           2:conv64@56_n32:20 2:conv128@28_n32:20 2:conv256@14_n32:20 2:conv512@7_n32:20 2:conv64@56_n1:20 2:conv512@7_n1:20 \
           3:conv5x5p2_96to256@27_n8:20 3:conv1x1_256to64@56_n8:20 5:conv128@28_n256:10 5:conv512@7_n8_coshard:20; do
   c=${cl%%:*}; r=${cl#*:}; l=${r%%:*}; it=${r#*:}
   run lane4x8 SMMC_LIB=paper_2411_15659_b200/lib/ab/lane8.so $c $l $it
   run main8x4 "" $c $l $it
 done
done
cat $O
