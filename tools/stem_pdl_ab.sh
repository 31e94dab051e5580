#!/bin/bash
# Programmatic dependent launch on the one-wave stem kernels: bench config 3
# and the VGG conv1_1 stem with and without SMMC_NO_PDL; stem parity tests first.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/stem_pdl; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stem.py -m gpu -q -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for v in pdl nopdl; do
  [ $v = nopdl ] && export SMMC_NO_PDL=1
  python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/cfg3_$v.json 2> $O/cfg3_$v.err
  python tools/n1_sweep.py --configs 3 --layers conv7x7s2p3_3to64@224_n8,conv11x11s4_3to96@227_n8 --cands "" > $O/sweep_$v.log 2>&1
done
python - <<'EOF'
import json
for v in ("pdl", "nopdl"):
    d = json.loads(open(f"gpurun_out/stem_pdl/cfg3_{v}.json").read().strip().splitlines()[-1])
    print(v, d["value"], [(l["layer"][:12], round(l["ms_avg"] * 1e3, 2), l["frac_fp32_peak"]) for l in d["layers"]])
    print(open(f"gpurun_out/stem_pdl/sweep_{v}.log").read()[:700])
EOF
