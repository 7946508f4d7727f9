#!/bin/bash
# Round-2 GPU session: parity tests + smoke, the default bench line (rmat20,
# e2e, cpu_baseline), the reference arm, bench lines of the other configs,
# the ncu launch list of the default bench command and an ncu --set full
# capture of its dominant kernel (k_hv_merge). Outputs under gpurun_out/$TAG.
TAG=${TAG:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
  echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/reference_default.json 2> $OUT/reference_default.err
for cm in ${RUNS:-stencil27_64:upper stencil27_64:precise uniform1m_k16:upper uniform1m_k16:precise amg_lap2048_agg2x2:upper amg_lap2048_agg2x2:precise uniform2k_k8:upper uniform2k_k8:precise}; do
  IFS=: read cfg mode <<< "$cm"
  timeout 600 python bench.py --config $cfg --mode $mode --steps 10 --warmup 3 --no-cpu-baseline \
    > $OUT/bench_${cfg}_${mode}.json 2> $OUT/bench_${cfg}_${mode}.err
done
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_hv_merge -c 1 -o $OUT/full_hv_merge \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
  ncu -i $OUT/full_hv_merge.ncu-rep --page raw --csv > $OUT/full_hv_merge.raw.csv 2>/dev/null
  ncu -i $OUT/full_hv_merge.ncu-rep --page details --csv > $OUT/full_hv_merge.details.csv 2>/dev/null
fi
du -sm $OUT > $OUT/size.txt
echo done > $OUT/DONE
