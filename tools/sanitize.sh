#!/bin/bash
# usage: tools/sanitize.sh <tool> [--only NAME]   (one tool per box call)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tool=$1; shift
CS=/usr/local/cuda/bin/compute-sanitizer
extra=""
[ "$tool" = "racecheck" ] && extra="--racecheck-report all"
timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 200 \
    python tools/sanitize_cases.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
echo "exit=$?" >> gpurun_out/sanitize_$tool.log
tail -5 gpurun_out/sanitize_$tool.log
