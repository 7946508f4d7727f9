#!/bin/bash
# Tuning experiment: rebuild libbrmerge.so with each variant's extra nvcc
# flags and run bench.py on the chosen configs; restores the default build.
# VARIANTS="name=flags;name=flags" (flags space-separated), outputs under
# gpurun_out/$TAG/var_<name>_<config>_<mode>.json
TAG=${TAG:-var}
OUT=gpurun_out/$TAG
mkdir -p $OUT
IFS=';' read -ra VS <<< "${VARIANTS:-default=}"
for v in "${VS[@]}"; do
  name=${v%%=*}; flags=${v#*=}
  BRM_NVCC_FLAGS="$flags" python -c "from paper_2206_06611_b200._build import build; build(force=True)" \
    > $OUT/build_$name.log 2>&1 || { echo "build $name failed" >> $OUT/errors.txt; continue; }
  for cfg in ${CONFIGS:-stencil27_64}; do
    for mode in ${MODES:-upper}; do
      timeout 600 python bench.py --config $cfg --mode $mode --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e \
        > $OUT/var_${name}_${cfg}_${mode}.json 2> $OUT/var_${name}_${cfg}_${mode}.err
    done
  done
done
python -c "from paper_2206_06611_b200._build import build; build(force=True)" > $OUT/build_restore.log 2>&1
echo done > $OUT/DONE
