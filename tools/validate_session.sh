#!/bin/bash
# Validation session at HEAD: parity tests, smoke, the default bench command
# (wall time recorded), the reference arm. Outputs under gpurun_out/$TAG.
TAG=${TAG:-r02g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q ) > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
( time timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err ) 2> $OUT/bench_default.time
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/reference_default.json 2> $OUT/reference_default.err ) 2> $OUT/reference_default.time
echo done > $OUT/DONE
