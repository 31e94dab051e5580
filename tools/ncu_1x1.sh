cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_1x1; mkdir -p $O
for cl in 5:conv1x1_64to256@56_n256 3:conv1x1_256to64@56_n8; do
  c=${cl%%:*}; l=${cl#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv1x1 -c 1 \
     -o $O/full_$l -f python tools/prof_layer.py --config $c --layer $l --iters 1 --graph 0 > $O/log_$l 2>&1
done
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/summary.txt 2>&1
for f in $O/full_*.ncu-rep; do ncu -i $f --page source --csv --print-source sass 2>/dev/null | head -c 3000000 > ${f%.ncu-rep}.sass.csv; done
rm -f $O/*.ncu-rep
cat $O/summary.txt
