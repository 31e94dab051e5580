#!/bin/bash
# Bounds-checked build of the library (SMMC_CHECKED: device asserts on every
# global/shared access of the kernels, see smmc_internal.cuh), selected at
# run time with SMMC_LIB=paper_2411_15659_b200/lib/checked/libsmmc.so.
cd "$(dirname "$0")/.."
python -m paper_2411_15659_b200.build --out paper_2411_15659_b200/lib/checked/libsmmc.so -DSMMC_CHECKED
