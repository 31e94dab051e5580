cd $GRAFT_REPO_ROOT
C="4,3,4,5 4,6,2,5 4,3,2,5 1,4,3,5 1,6,2,5;4,5,4,5 4,6,2,5 4,9,2,5 4,11,2,5 4,5,4 1,8,2,5;4,9,4,5 4,8,4,5 4,18,2,5 4,16,2,5 3,18,2,5 1,16,2,5;4,18,4,5 4,16,4,5 4,32,2,5 4,24,2,5 3,32,2,5 3,18,2,5"
L=conv64@56_n1,conv128@28_n1,conv256@14_n1,conv512@7_n1
python tools/n1_sweep.py --configs 2 --layers $L --cands "$C" > gpurun_out/n1_sweep2.log 2>&1
SMMC_NO_PDL=1 python tools/n1_sweep.py --configs 2 --layers $L --cands "$C" > gpurun_out/n1_sweep2_nopdl.log 2>&1
export SMMC_LIB=$PWD/paper_2411_15659_b200/lib/ab/tl.so
run() { SMMC_FORCE_PLAN=$2 python tools/timeline_probe.py --cold 0 --config 2 --layer $1; }
{ run conv64@56_n1 4,3,4,5; run conv64@56_n1 4,6,2,5; run conv512@7_n1 4,18,4,5; } > gpurun_out/n1_tl3.log 2>&1
