#!/bin/bash
# Re-entry validation in one box session: GPU tests, smoke, default bench, reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/reentry; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
tail -3 $O/gputests.log; tail -2 $O/smoke.log; cat $O/bench.json | cut -c1-600; cat $O/bench_ref.json | cut -c1-400
