#!/bin/bash
# Session: parity + smoke at HEAD, default line, heavy ILP variants.
OUT=gpurun_out/s3
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
TAG=s3 VARIANTS="ilp1=-DBRM_HV_ILP=1;ilp2=-DBRM_HV_ILP=2;ilp3=-DBRM_HV_ILP=3" CONFIGS=rmat20_ef16 MODES=precise STEPS=5 bash tools/variants.sh
echo done > $OUT/DONE
