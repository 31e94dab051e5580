cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_1x1; mkdir -p $O
for env in "SMMC_1X1_WRES=1" "SMMC_1X1_WRES=0"; do
  tag=${env#*=}
  env $env timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv1x1 -c 1 \
     -o $O/full_wres$tag -f python tools/prof_layer.py --config 5 --layer conv1x1_64to256@56_n256 --iters 1 --graph 0 > $O/log$tag 2>&1
done
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/summary.txt 2>&1
for f in $O/full_*.ncu-rep; do ncu -i $f --page raw --csv 2>/dev/null > ${f%.ncu-rep}.raw.csv; done
rm -f $O/*.ncu-rep
