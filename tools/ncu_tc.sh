cd $GRAFT_REPO_ROOT
O=gpurun_out/tc_ncu; mkdir -p $O
for l in conv64@56_n32 conv128@28_n32 conv256@14_n32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv_tc|pack_input" -c 2 \
     -o $O/full_$l -f python tools/prof_layer.py --config 2 --layer $l --iters 1 --graph 0 --mode bf16x3_tc > $O/full_$l.log 2>&1
done
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/summary.txt 2>&1
for f in $O/full_*.ncu-rep; do ncu -i $f --page raw --csv 2>/dev/null > ${f%.ncu-rep}.raw.csv; done
rm -f $O/*.ncu-rep
