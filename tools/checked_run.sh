#!/bin/bash
# Run the kernel-family cases and the GPU test suite against the bounds-checked
# library (tools/checked_build.sh); logs under gpurun_out/checked_*.log
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export SMMC_LIB=$PWD/paper_2411_15659_b200/lib/checked/libsmmc.so
timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo "exit=$?" >> gpurun_out/checked_cases.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_gputests.log 2>&1; echo "exit=$?" >> gpurun_out/checked_gputests.log
