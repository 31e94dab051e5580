cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
SMMC_LIB=$PWD/paper_2411_15659_b200/lib/ab/legacy_memset.so python -m pytest tests/test_gpu_robustness.py -q -p no:cacheprovider -k "fresh_process or weight_heavy" 2>&1 | tail -3
done > gpurun_out/race_memset_legacy.log
for i in 1 2 3; do
python -m pytest tests/test_gpu_robustness.py -q -p no:cacheprovider -k "fresh_process or weight_heavy" 2>&1 | tail -3
done > gpurun_out/race_memset_fixed.log
