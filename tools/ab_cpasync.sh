#!/bin/bash
# Same-box A/B of k_hv_merge's gather: synchronous batched loads (default)
# vs cp.async (BRM_HV_CPASYNC=1): bench line + ncu warp-state stalls of one
# k_hv_merge launch for each. Outputs under gpurun_out/$TAG.
TAG=${TAG:-ab_cpasync}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for v in sync:"" cpasync:"-DBRM_HV_CPASYNC=1"; do
  name=${v%%:*}; flags=${v#*:}
  BRM_NVCC_FLAGS="$flags" python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build_$name.log 2>&1
  [ "${SKIP_BENCH:-0}" = 1 ] || timeout 900 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/bench_$name.json 2> $OUT/bench_$name.err
  timeout 1500 ncu --section WarpStateStats --section SchedulerStats --section SpeedOfLight --section MemoryWorkloadAnalysis \
    --clock-control none -k regex:k_hv_merge -c 1 -o $OUT/ncu_$name python tools/prof_one.py > $OUT/ncu_$name.log 2>&1
  ncu -i $OUT/ncu_$name.ncu-rep --page raw --csv > $OUT/ncu_$name.raw.csv 2>/dev/null
  ncu -i $OUT/ncu_$name.ncu-rep --page details --csv > $OUT/ncu_$name.details.csv 2>/dev/null
  rm -f $OUT/ncu_$name.ncu-rep
done
python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build_restore.log 2>&1
echo done > $OUT/DONE
