#!/bin/bash
# One box session: every bench config (fp32 + bf16 variant), the ncu launch
# list of the default bench, and --set full captures of the top kernels.
set -u
mkdir -p gpurun_out
STEPS=${STEPS:-10} CPU_S=${CPU_S:-5} bash tools/run_all_configs.sh
for c in 2 5; do
  timeout 900 python bench.py --config $c --mode bf16_tc --steps 10 --warmup 3 --cpu-seconds 5 \
     --details gpurun_out/bench_tc_cfg$c.json > gpurun_out/bench_tc_cfg$c.log 2>&1
  echo "tc config $c rc=$?"
  timeout 900 python bench.py --config $c --mode bf16x3_tc --steps 10 --warmup 3 --cpu-seconds 5 \
     --details gpurun_out/bench_tc3_cfg$c.json > gpurun_out/bench_tc3_cfg$c.log 2>&1
  echo "tc3 config $c rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-e2e \
   --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
for l in conv512@7_n32 conv64@56_n32 conv128@28_n32 conv256@14_n32 conv64@56_n1; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_ffma -c 1 \
     -o gpurun_out/full_$l -f python tools/prof_layer.py --config 2 --layer $l --iters 1 --graph 0 \
     > gpurun_out/full_$l.log 2>&1
  echo "ncu $l rc=$?"
done
for l in conv256@14_n256 conv1x1_64to256@56_n256 conv128@28_n256; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 \
     -o gpurun_out/full_tc_$l -f python tools/prof_layer.py --config 5 --layer $l --iters 1 \
     --graph 0 --mode bf16_tc > gpurun_out/full_tc_$l.log 2>&1
  echo "ncu tc $l rc=$?"
done
for l in conv256@14_n256 conv128@28_n256; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv_tc|pack_input" -c 2 \
     -o gpurun_out/full_tc3_$l -f python tools/prof_layer.py --config 5 --layer $l --iters 1 \
     --graph 0 --mode bf16x3_tc > gpurun_out/full_tc3_$l.log 2>&1
  echo "ncu tc3 $l rc=$?"
done
# summaries on the box (the .ncu-rep files exceed what gpurun copies back)
python tools/ncu_summary.py gpurun_out/full_*.ncu-rep > gpurun_out/ncu_summaries.txt 2>&1
python tools/ncu_traffic.py gpurun_out/traffic.json gpurun_out/full_conv*.ncu-rep > gpurun_out/traffic.log 2>&1
mkdir -p gpurun_out/reps && mv gpurun_out/full_conv512@7_n32.ncu-rep gpurun_out/reps/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
