#!/bin/bash
# Driver-style validation in one box session: GPU tests, smoke, default bench,
# reference arm, the bounds-checked build over all kernel families + suite.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
export SMMC_LIB=$PWD/paper_2411_15659_b200/lib/checked/libsmmc.so
timeout 900 python tools/sanitize_cases.py > $O/checked_cases.log 2>&1; echo "exit=$?" >> $O/checked_cases.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/checked_gputests.log 2>&1; echo "exit=$?" >> $O/checked_gputests.log
