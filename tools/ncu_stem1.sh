cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_ncu; mkdir -p $O
l=vgg01_3to64@224_n64
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_stem -c 1 \
   -o $O/full_$l -f python tools/prof_layer.py --config 4 --layer $l --iters 1 --graph 0 > $O/full_$l.log 2>&1
python tools/ncu_summary.py $O/full_$l.ncu-rep > $O/summary_rw.txt 2>&1
ncu -i $O/full_$l.ncu-rep --page source --csv --print-source sass 2>/dev/null | head -c 3000000 > $O/full_$l.sass.csv
rm -f $O/*.ncu-rep
cat $O/summary_rw.txt
