#!/bin/bash
# Round-2 profile session: default bench (config 4) + reference arm, every
# config's fp32 line, the bf16 lines (pack timed), the ncu launch list of the
# default bench and --set full captures of its dominant kernels.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
O=gpurun_out/prof
timeout 900 python bench.py --details $O/bench_default.details.json > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for c in 1 2 3 5; do
  timeout 900 python bench.py --config $c --cpu-seconds 4 --details $O/bench_cfg$c.details.json > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
for c in 2 5; do
  for m in bf16_tc bf16_tc_prepacked bf16x3_tc; do
    timeout 900 python bench.py --config $c --mode $m --steps 10 --warmup 3 --no-cpu-baseline \
      --details $O/bench_${m}_cfg$c.details.json > $O/bench_${m}_cfg$c.json 2> $O/bench_${m}_cfg$c.err
  done
done
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/b_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
   --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-e2e \
   --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?" >> $O/ncu_launch.log
for l in vgg02_64to64@224_n64 vgg09_512to512@28_n64 vgg06_256to256@56_n64 vgg01_3to64@224_n64; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv_" -c 1 \
     -o $O/full_$l -f python tools/prof_layer.py --config 4 --layer $l --iters 1 --graph 0 \
     > $O/full_$l.log 2>&1
  echo "ncu $l rc=$?" >> $O/ncu_launch.log
done
for cl in 5:conv1x1_64to256@56_n256 3:conv7x7s2p3_3to64@224_n8 3:conv11x11s4_3to96@227_n8 3:conv1x1_256to64@56_n8; do
  c=${cl%%:*}; l=${cl#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv" -c 1 \
     -o $O/full_$l -f python tools/prof_layer.py --config $c --layer $l --iters 1 --graph 0 \
     > $O/full_$l.log 2>&1
  echo "ncu $l rc=$?" >> $O/ncu_launch.log
done
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/ncu_summaries.txt 2>&1
python tools/ncu_traffic.py $O/traffic.json $O/full_*.ncu-rep > $O/traffic.log 2>&1
rm -f $O/*.ncu-rep
