#!/bin/bash
# A/B session: GPU parity tests on the default build, then bench lines of
# VARIANTS (tools/variants.sh) on CONFIGS x MODES. Outputs under gpurun_out/$TAG.
TAG=${TAG:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
TAG=$TAG bash tools/variants.sh
echo done > $OUT/DONE
