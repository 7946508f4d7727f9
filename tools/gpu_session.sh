#!/bin/bash
# One GPU session: parity tests, bench on every config, ncu launch list and a
# full capture of the dominant kernel. Outputs under gpurun_out/$TAG/.
TAG=${TAG:-s1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
for cfg in ${CONFIGS:-stencil27_64 uniform2k_k8 uniform1m_k16 rmat20_ef16 amg_lap2048_agg2x2}; do
  for mode in ${MODES:-precise upper}; do
    timeout 600 python bench.py --config $cfg --mode $mode --steps ${STEPS:-10} --warmup 3 > $OUT/bench_${cfg}_${mode}.json 2> $OUT/bench_${cfg}_${mode}.err
  done
done
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tier -c ${NCU_COUNT:-4} -o $OUT/full \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
fi
echo done > $OUT/DONE
