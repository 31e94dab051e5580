#!/bin/bash
# all BASELINE configs' bench lines (fp32 product) + GPU tests; logs in gpurun_out/
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
for c in ${CONFIGS:-1 2 3 5 4}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS} --details gpurun_out/bench_cfg$c.details.json > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
