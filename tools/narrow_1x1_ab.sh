#!/bin/bash
# A/B of the warp-tile 1x1 kernel (c_o <= 64) against the tile kernels on the
# config-3 1x1 256->64 N=8 layer; parity tests first.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/narrow; mkdir -p $O; rm -f $O/ab.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "persistent_1x1" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -5 $O/tests.log
run() { echo "== $*" >> $O/ab.log; env "$@" timeout 600 python tools/n1_sweep.py --configs 3 --layers conv1x1_256to64@56_n8 --cands "4,1,2" >> $O/ab.log 2>&1; }
run SMMC_1X1_NARROW=1
run SMMC_1X1_NARROW=1 SMMC_NO_PDL=1
run SMMC_1X1_NARROW=0
cat $O/ab.log
