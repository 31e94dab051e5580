cd $GRAFT_REPO_ROOT
for rep in 1 2; do for env in "" "SMMC_NO_PDL=1"; do echo "== $env"
for l in conv64@56_n1 conv128@28_n1 conv256@14_n1 conv512@7_n1; do env $env python tools/prof_layer.py --config 2 --layer $l --iters 20; done
env $env python tools/prof_layer.py --config 5 --layer conv512@7_n8_coshard --iters 20
done; done > gpurun_out/n1_pdl_ab.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputests.log 2>&1
for c in 1 2; do python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bt_cfg$c.json 2>gpurun_out/bt_cfg$c.err; done
