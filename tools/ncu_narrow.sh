cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_narrow; mkdir -p $O
l=conv1x1_256to64@56_n8
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv1x1 -c 1 \
   -o $O/full_$l -f python tools/prof_layer.py --config 3 --layer $l --iters 1 --graph 0 > $O/log_$l 2>&1
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/summary.txt 2>&1
for f in $O/full_*.ncu-rep; do ncu -i $f --page source --csv --print-source sass 2>/dev/null | head -c 3000000 > ${f%.ncu-rep}.sass.csv; done
rm -f $O/*.ncu-rep
cat $O/summary.txt
