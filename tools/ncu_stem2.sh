cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_ncu; mkdir -p $O
l=conv7x7s2p3_3to64@224_n8
export SMMC_LIB=$PWD/paper_2411_15659_b200/lib/ab/m2a.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_stem -c 1 \
   -o $O/ring_$l -f python tools/prof_layer.py --config 3 --layer $l --iters 1 --graph 0 > $O/ring_$l.log 2>&1
python tools/ncu_summary.py $O/ring_$l.ncu-rep > $O/summary_ring.txt 2>&1
ncu -i $O/ring_$l.ncu-rep --page source --csv --print-source sass 2>/dev/null | head -c 3000000 > $O/ring_$l.sass.csv
rm -f $O/*.ncu-rep
cat $O/summary_ring.txt
