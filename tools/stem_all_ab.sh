# the three BASELINE stems: round-1 kernel (SMMC_STEM_RW0 for conv1_1) vs main; stem parity tests first,
# then the stem tests against the bounds-checked library
cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_all_ab.log
python -m pytest tests/test_gpu_stem.py -q -x -p no:cacheprovider > $O 2>&1
SMMC_LIB=$PWD/paper_2411_15659_b200/lib/checked/libsmmc.so python -m pytest tests/test_gpu_stem.py -q -x -p no:cacheprovider >> $O 2>&1
for rep in 1 2; do
  python tools/prof_layer.py --config 4 --layer vgg01_3to64@224_n64 --iters 20 | tail -1
  python tools/prof_layer.py --config 3 --layer conv7x7s2p3_3to64@224_n8 --iters 20 | tail -1
  python tools/prof_layer.py --config 3 --layer conv11x11s4_3to96@227_n8 --iters 20 | tail -1
done >> $O 2>&1
cat $O
