cd $GRAFT_REPO_ROOT
for l in conv64@56_n1 conv128@28_n1 conv256@14_n1 conv512@7_n1; do
  python tools/prof_layer.py --config 2 --layer $l --iters 50
  python tools/prof_layer.py --config 2 --layer $l --iters 50 --graph 0
done > gpurun_out/n1_times.log 2>&1
SMMC_LIB=$PWD/paper_2411_15659_b200/lib/ab/tl.so python tools/timeline_probe.py --config 2 --layer conv64@56_n1 --layer conv128@28_n1 --layer conv256@14_n1 --layer conv512@7_n1 > gpurun_out/n1_tl_cold.log 2>&1
SMMC_LIB=$PWD/paper_2411_15659_b200/lib/ab/tl.so python tools/timeline_probe.py --cold 0 --config 2 --layer conv64@56_n1 --layer conv128@28_n1 --layer conv256@14_n1 --layer conv512@7_n1 > gpurun_out/n1_tl_warm.log 2>&1
timeout 900 python tools/sanitize_cases.py --repeat 200 --noise > gpurun_out/race_hunt.log 2>&1; echo "exit=$?" >> gpurun_out/race_hunt.log
