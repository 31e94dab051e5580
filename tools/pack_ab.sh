cd $GRAFT_REPO_ROOT
for rep in 1 2; do for env in "" "SMMC_PACK_TILES=1"; do echo "== $env"
for l in conv64@56_n32 conv128@28_n32 conv256@14_n32 conv512@7_n32; do
 env $env python tools/prof_layer.py --config 2 --layer $l --iters 20 --mode bf16x3_tc; done; done; done > gpurun_out/pack_ab.log 2>&1
python -m pytest tests/test_gpu_tc.py tests/test_gpu_tc3.py -q -p no:cacheprovider >> gpurun_out/pack_ab.log 2>&1
