#!/bin/bash
# One GPU session: parity tests, bench on the chosen configs, and (only if
# the tests and the plain bench passed) an ncu launch list + full capture of
# the merge kernels. Outputs under gpurun_out/$TAG/.
TAG=${TAG:-s1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
ok=1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; rc=$?
  echo "pytest rc=$rc" >> $OUT/pytest_gpu.log; [ $rc = 0 ] || ok=0
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; rc=$?
  echo "smoke rc=$rc" >> $OUT/smoke.log; [ $rc = 0 ] || ok=0
fi
for cfg in ${CONFIGS:-stencil27_64 uniform1m_k16 amg_lap2048_agg2x2}; do
  for mode in ${MODES:-upper precise}; do
    timeout 900 python bench.py --config $cfg --mode $mode --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} \
      > $OUT/bench_${cfg}_${mode}.json 2> $OUT/bench_${cfg}_${mode}.err || ok=0
  done
done
if [ "${NCU:-1}" = 1 ] && [ $ok = 1 ]; then
  NCFG=${NCU_CONFIG:-stencil27_64}; NMODE=${NCU_MODE:-upper}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --config $NCFG --mode $NMODE --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_tier} -c ${NCU_COUNT:-6} -o $OUT/full \
    python bench.py --config $NCFG --mode $NMODE --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
  for extra in ${NCU_EXTRA:-}; do  # config:mode:kernel-regex
    IFS=: read ECFG EMODE EKER <<< "$extra"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$EKER -c ${NCU_COUNT:-6} -o $OUT/full_$ECFG \
      python bench.py --config $ECFG --mode $EMODE --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_$ECFG.log 2>&1
  done
else
  echo "ncu skipped (ok=$ok)" > $OUT/ncu_skipped.txt
fi
echo done > $OUT/DONE
