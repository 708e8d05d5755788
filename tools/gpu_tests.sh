#!/bin/bash
# gpurun -- bash tools/gpu_tests.sh TAG [pytest selection...]: GPU tests + one bench line.
TAG=${1:-x}; shift
SEL=${@:-tests}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
timeout 2400 python -m pytest $SEL -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -15 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
tail -3 $OUT/bench_$TAG.err
echo done
