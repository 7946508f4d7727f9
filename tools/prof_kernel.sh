#!/bin/bash
# ncu --set full of one kernel (regex K) on CFG/MODE, raw + source (cuda,sass)
# + details pages. Optional BRM_NVCC_FLAGS rebuild. Outputs under gpurun_out/$TAG.
TAG=${TAG:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
BRM_NVCC_FLAGS="${FLAGS:-}" python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build.log 2>&1
for spec in ${SPECS:-stencil27_64:upper:k_wtier}; do
  IFS=: read CFG MODE K <<< "$spec"
  N=${CFG}_${MODE}_${TAGK:-$(echo $K | tr -c "a-zA-Z0-9_\n" _)}
  timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -c 1 -o $OUT/$N \
    python tools/prof_one.py --config $CFG --mode $MODE > $OUT/ncu_$N.log 2>&1
  ncu -i $OUT/$N.ncu-rep --page raw --csv > $OUT/$N.raw.csv 2>/dev/null
  ncu -i $OUT/$N.ncu-rep --page source --csv --print-source cuda,sass > $OUT/$N.source.csv 2>/dev/null
  ncu -i $OUT/$N.ncu-rep --page details --csv > $OUT/$N.details.csv 2>/dev/null
done
python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build_restore.log 2>&1
echo done > $OUT/DONE
