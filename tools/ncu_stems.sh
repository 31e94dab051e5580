cd $GRAFT_REPO_ROOT
O=gpurun_out/stem_ncu; mkdir -p $O
for cl in 4:vgg01_3to64@224_n64 3:conv7x7s2p3_3to64@224_n8 3:conv11x11s4_3to96@227_n8; do
  c=${cl%%:*}; l=${cl#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_stem -c 1 \
     -o $O/full_$l -f python tools/prof_layer.py --config $c --layer $l --iters 1 --graph 0 > $O/full_$l.log 2>&1
done
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/summary.txt 2>&1
for f in $O/full_*.ncu-rep; do ncu -i $f --page source --csv --print-source sass 2>/dev/null | head -c 3000000 > ${f%.ncu-rep}.sass.csv; done
rm -f $O/*.ncu-rep
