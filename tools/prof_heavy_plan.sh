OUT=gpurun_out/r02e_prof
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_hv_plan -c 1 -o $OUT/plan1 python tools/prof_one.py --config rmat20_ef16 --mode precise > $OUT/ncu_plan1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_hv_merge --launch-skip 1 -c 1 -o $OUT/merge_lvl1 python tools/prof_one.py --config rmat20_ef16 --mode precise > $OUT/ncu_merge_lvl1.log 2>&1
for N in plan1 merge_lvl1; do
  ncu -i $OUT/$N.ncu-rep --page raw --csv > $OUT/$N.raw.csv 2>/dev/null
  ncu -i $OUT/$N.ncu-rep --page source --csv --print-source cuda,sass > $OUT/$N.source.csv 2>/dev/null
done
rm -f $OUT/*.ncu-rep
echo done > $OUT/DONE
