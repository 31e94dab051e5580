# A/B of the resident-window stem kernel (conv1_1) against the round-1 stem
# kernel and the RW1_ tile variants of tools/stem_rw_variants.py (each variant
# first runs the resident-window parity tests).
cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_rw_ab.log
python -m pytest tests/test_gpu_stem.py -q -x -p no:cacheprovider > $O 2>&1
for v in paper_2411_15659_b200/lib/ab/rw_*.so; do
  echo "== tests $v" >> $O
  SMMC_LIB=$v python -m pytest tests/test_gpu_stem.py -q -x -p no:cacheprovider -k "resident" 2>&1 | tail -3 >> $O
done
for rep in 1 2; do
  echo "== round-1 kernel"; SMMC_STEM_RW0=1 python tools/prof_layer.py --config 4 --layer vgg01_3to64@224_n64 --iters 20 | tail -1
  echo "== main"; python tools/prof_layer.py --config 4 --layer vgg01_3to64@224_n64 --iters 20 | tail -1
  for v in paper_2411_15659_b200/lib/ab/rw_*.so; do
    echo "== $v"; SMMC_LIB=$v python tools/prof_layer.py --config 4 --layer vgg01_3to64@224_n64 --iters 20 | tail -1
  done
done >> $O 2>&1
cat $O
