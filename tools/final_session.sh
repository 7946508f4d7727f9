#!/bin/bash
# Round-end GPU session: parity tests + smoke, bench lines for every config
# and mode, ncu launch list of the default workload, ncu --set full captures
# of the dominant kernels, the rmat20 line, the default bench line and the
# reference arm. Keeps gpurun_out/$TAG under the 64 MiB copy-back limit by
# exporting each capture's raw page to CSV and dropping large reports.
TAG=${TAG:-final}
OUT=gpurun_out/$TAG
TAG=$TAG CONFIGS="stencil27_64 uniform1m_k16 amg_lap2048_agg2x2 uniform2k_k8" MODES="upper precise" NCU_COUNT=${NCU_COUNT:-2} \
  NCU_EXTRA="uniform1m_k16:upper:k_tier amg_lap2048_agg2x2:precise:k_tiny rmat20_ef16:precise:k_slab2" bash tools/gpu_session.sh
timeout 900 python bench.py --config rmat20_ef16 --mode precise --steps 5 --warmup 3 > $OUT/bench_rmat20_ef16_precise.json 2> $OUT/bench_rmat20_ef16_precise.err
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --impl reference > $OUT/reference_default.json 2> $OUT/reference_default.err
for r in $OUT/*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
done
ncu -i $OUT/full.ncu-rep --page source --csv --print-source cuda,sass > $OUT/full.source.csv 2>/dev/null
gzip -f $OUT/full.source.csv
for r in $(ls -S $OUT/*.ncu-rep 2>/dev/null); do
  [ $(du -sm $OUT | cut -f1) -gt 56 ] && rm -f "$r"
done
du -sm $OUT > $OUT/size.txt
