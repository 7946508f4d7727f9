#!/bin/bash
# Quick GPU check: build, parity tests (optionally a -k filter), then bench
# lines for "config:mode" pairs. Outputs under gpurun_out/$TAG/.
TAG=${TAG:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
for cm in ${RUNS:-stencil27_64:upper}; do
  IFS=: read cfg mode <<< "$cm"
  timeout 900 python bench.py --config $cfg --mode $mode --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline --no-e2e} \
    > $OUT/bench_${cfg}_${mode}.json 2> $OUT/bench_${cfg}_${mode}.err
done
echo done > $OUT/DONE
