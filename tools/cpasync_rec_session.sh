#!/bin/bash
# Round-2 session: GPU tests at HEAD; same-box A/B of cp.async staging in the
# block-per-row tiers (5-6) on rmat20 (bench lines + ncu of the tier-6
# numeric launch under both builds); GPU tests on the cp.async build too.
OUT=gpurun_out/cpa
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for v in sync:"" cpasync:"-DBRM_REC_CPASYNC=1"; do
  name=${v%%:*}; flags=${v#*:}
  BRM_NVCC_FLAGS="$flags" python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build_$name.log 2>&1
  if [ $name = cpasync ]; then
    timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size" > $OUT/pytest_gpu_$name.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$name.log
  fi
  timeout 900 python bench.py --config rmat20_ef16 --mode precise --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_$name.json 2> $OUT/bench_$name.err
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_tierILi256ELi6656 -c 1 -o $OUT/t6_$name \
    python tools/prof_one.py --config rmat20_ef16 --mode precise > $OUT/ncu_t6_$name.log 2>&1
  ncu -i $OUT/t6_$name.ncu-rep --page raw --csv > $OUT/t6_$name.raw.csv 2>/dev/null
done
python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build_restore.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
echo done > $OUT/DONE
