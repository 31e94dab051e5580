cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for env in "" "SMMC_STEM_PERSIST0=1" "SMMC_STEM_PERSIST0=1 SMMC_STEM_CI0=1"; do
  echo "== $env"
  env $env python tools/prof_layer.py --config 4 --layer vgg01_3to64@224_n64 --iters 20
  env $env python tools/prof_layer.py --config 3 --layer conv7x7s2p3_3to64@224_n8 --iters 20
  env $env python tools/prof_layer.py --config 3 --layer conv11x11s4_3to96@227_n8 --iters 20
done
done > gpurun_out/stem_persist_ab.log 2>&1
python -m pytest tests/test_gpu_stem.py -q -p no:cacheprovider >> gpurun_out/stem_persist_ab.log 2>&1
