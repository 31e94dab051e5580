cd $GRAFT_REPO_ROOT
for rep in 1 2; do for env in "" "SMMC_1X1_WRES=0"; do echo "== $env"
 env $env python tools/prof_layer.py --config 5 --layer conv1x1_64to256@56_n256 --iters 10
 env $env SMMC_FORCE_PLAN= python tools/prof_layer.py --config 3 --layer conv1x1_256to64@56_n8 --iters 20
done; done > gpurun_out/wres_ab.log 2>&1
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "1x1" >> gpurun_out/wres_ab.log 2>&1
