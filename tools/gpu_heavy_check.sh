#!/bin/bash
# GPU check of the heavy-row path: focused parity tests, then rmat20 lines.
TAG=${TAG:-hv}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:--k "heavy or slab or empty_lists or workload_shapes or recursive or pairing or tier_boundaries"} > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
for cm in ${RUNS:-rmat20_ef16:precise}; do
  IFS=: read cfg mode <<< "$cm"
  timeout 900 python bench.py --config $cfg --mode $mode --steps ${STEPS:-5} --warmup 2 ${BENCH_ARGS:---no-cpu-baseline --no-e2e} \
    > $OUT/bench_${cfg}_${mode}.json 2> $OUT/bench_${cfg}_${mode}.err
done
echo done > $OUT/DONE
