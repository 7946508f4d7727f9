#!/bin/bash
# ncu captures of one config: launch list + --set full of selected kernels.
TAG=${TAG:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CFG=${CFG:-rmat20_ef16}
MODE=${MODE:-precise}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/prof_one.py --config $CFG --mode $MODE > $OUT/run.log 2>&1
echo "run rc=$?" >> $OUT/run.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python tools/prof_one.py --config $CFG --mode $MODE > $OUT/ncu_launch.log 2>&1
for K in ${KERNELS:-k_hv_merge k_hv_plan}; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o $OUT/full_$K \
    python tools/prof_one.py --config $CFG --mode $MODE > $OUT/ncu_full_$K.log 2>&1
  ncu -i $OUT/full_$K.ncu-rep --page raw --csv > $OUT/full_$K.raw.csv 2>/dev/null
  ncu -i $OUT/full_$K.ncu-rep --page source --csv > $OUT/full_$K.source.csv 2>/dev/null
  ncu -i $OUT/full_$K.ncu-rep --page details --csv > $OUT/full_$K.details.csv 2>/dev/null
done
echo done > $OUT/DONE
