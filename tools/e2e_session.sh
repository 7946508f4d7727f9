OUT=gpurun_out/${TAG:-e2e1}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "host" > $OUT/pytest_host.log 2>&1; echo "rc=$?" >> $OUT/pytest_host.log
timeout 1200 python bench.py --no-cpu-baseline > $OUT/bench_rmat20.json 2> $OUT/bench_rmat20.err
for c in stencil27_64:upper uniform1m_k16:upper amg_lap2048_agg2x2:precise; do IFS=: read cfg mode <<< "$c"
timeout 600 python bench.py --config $cfg --mode $mode --no-cpu-baseline > $OUT/bench_${cfg}.json 2> $OUT/bench_${cfg}.err; done
