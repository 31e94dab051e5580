cd $GRAFT_REPO_ROOT
export SMMC_LIB=$PWD/paper_2411_15659_b200/lib/ab/tl.so
run() { SMMC_FORCE_PLAN=$2 python tools/timeline_probe.py --cold 0 --config 2 --layer $1; }
{ run conv64@56_n1 4,3,4,5; run conv64@56_n1 1,4,3; run conv512@7_n1 4,18,4,5; run conv128@28_n1 4,5,4; } > gpurun_out/n1_tl4.log 2>&1
unset SMMC_LIB
python tools/n1_sweep.py --configs 2 --layers conv64@56_n1,conv128@28_n1,conv256@14_n1,conv512@7_n1 --cands "4,3,4,5 4,3,2,5;4,5,4 4,5,4,5;4,9,4,5 1,16,2,5;4,18,4,5 4,16,4,5" > gpurun_out/n1_sweep3.log 2>&1
