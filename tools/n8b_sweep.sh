cd $GRAFT_REPO_ROOT
python tools/n1_sweep.py --configs 3,2 --layers conv5x5p2_96to256@27_n8,conv512@7_n32,conv256@14_n32 --cands \
 "3,3,1,5 3,2,2,5 1,3,1,5 0,4,1,5 3,4 3,3 1,4 0,3 3,2,1,5;3,0 3,2,2,5 1,3,1,5 0,4,1,5 3,3,1,5 4,2,2,5 3,4,1,5 0,2,1,5;0,3 0,2,1,5 1,2,2,5 3,3,1,5 0,3,1,5 3,2,2,5 1,3,1,5" --iters 10 > gpurun_out/n8b_sweep.log 2>&1
