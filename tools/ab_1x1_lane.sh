cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_1x1_lane.log; : > $O
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "1x1 or wres or persistent" 2>&1 | tail -2 >> $O
run() { echo -n "$1 " >> $O; env $2 python tools/prof_layer.py --config $3 --layer $4 --iters 20 2>&1 | tail -1 >> $O; }
for rep in 1 2; do
 L=conv1x1_64to256@56_n256
 run lane4x8 SMMC_LIB=paper_2411_15659_b200/lib/ab/lane8.so 5 $L
 run main "" 5 $L
 run main_streamed SMMC_1X1_WRES=0 5 $L
 L=conv1x1_256to64@56_n8
 run main "" 3 $L

done
cat $O
