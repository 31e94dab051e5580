cd $GRAFT_REPO_ROOT
python tools/n1_sweep.py --configs 2 --layers conv64@56_n1,conv128@28_n1,conv256@14_n1,conv512@7_n1 --cands \
 "4,3,4 4,3,4,5 4,6,2 4,6,2,5 4,4,4;4,5,4 4,5,4,5 4,4,4 4,8,2;4,8,4 4,9,4,5 4,8,2 4,6,4;4,8,4 4,18,4,5 4,16,4,5 4,8,2" > gpurun_out/n1_sweep4.log 2>&1
