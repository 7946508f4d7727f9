#!/bin/bash
# Round-2 closing session: parity + smoke, the default bench line (rmat20,
# e2e, cpu_baseline), the reference arm (default config and the stencil's
# whole matrix), every config and mode, the ncu launch list of the default
# bench command, ncu --set full of each config's dominant kernel, and the
# one-GPU per-block scaling emulation. Outputs under gpurun_out/$TAG.
TAG=${TAG:-r02f}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/reference_default.json 2> $OUT/reference_default.err
timeout 900 python bench.py --impl reference --config stencil27_64 --steps 3 --warmup 1 > $OUT/reference_stencil27_64.json 2> $OUT/reference_stencil27_64.err
for cm in stencil27_64:upper stencil27_64:precise uniform1m_k16:upper uniform1m_k16:precise amg_lap2048_agg2x2:upper amg_lap2048_agg2x2:precise uniform2k_k8:upper uniform2k_k8:precise; do
  IFS=: read cfg mode <<< "$cm"
  timeout 600 python bench.py --config $cfg --mode $mode --steps 10 --warmup 3 --no-cpu-baseline \
    > $OUT/bench_${cfg}_${mode}.json 2> $OUT/bench_${cfg}_${mode}.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
for spec in rmat20_ef16:precise:k_hv_merge:full_hv_merge stencil27_64:upper:k_tierILi32ELi768:full_stencil_t4 uniform1m_k16:upper:k_tierILi32ELi256:full_uniform_t3 amg_lap2048_agg2x2:precise:k_tinyILb1ELi2:full_amg_t1; do
  IFS=: read cfg mode K N <<< "$spec"
  timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -c 1 -o $OUT/$N \
    python bench.py --config $cfg --mode $mode --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_$N.log 2>&1
  ncu -i $OUT/$N.ncu-rep --page raw --csv > $OUT/$N.raw.csv 2>/dev/null
  ncu -i $OUT/$N.ncu-rep --page details --csv > $OUT/$N.details.csv 2>/dev/null
  ncu -i $OUT/$N.ncu-rep --page source --csv --print-source cuda,sass > $OUT/$N.source.csv 2>/dev/null
done
timeout 1500 python tools/scale_emulate.py --config rmat20_ef16 > $OUT/scale_rmat20.json 2> $OUT/scale_rmat20.err
timeout 600 python tools/scale_emulate.py --config amg_lap2048_agg2x2 > $OUT/scale_amg.json 2> $OUT/scale_amg.err
rm -f $OUT/*.ncu-rep.tmp
du -sm $OUT > $OUT/size.txt
echo done > $OUT/DONE
