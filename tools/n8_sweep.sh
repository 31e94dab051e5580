cd $GRAFT_REPO_ROOT
python tools/n1_sweep.py --configs 3,5 --layers conv1x1_256to64@56_n8,conv512@7_n8_coshard --cands \
 "1,3 1,3,1,5 1,2 1,4 4,2,1,5 4,3,1,5 4,2,2,5 4,1,2 4,1,4 3,2 0,2;3,24 4,5,2,5 4,5,4,5 4,9,2,5 0,9,1,5 3,10,1,5 3,5,2,5 1,8,2,5 1,9,1,5 3,20,1,5 4,10,2,5" > gpurun_out/n8_sweep.log 2>&1
