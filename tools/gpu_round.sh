#!/bin/bash
# One gpurun call: GPU tests, smoke, bench line, ncu launch list and full
# captures of K1 and of one projection GEMM. Usage: gpurun -- bash tools/gpu_round.sh TAG [quick]
TAG=${1:-r01}
MODE=${2:-full}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
if [ "$MODE" = "full" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
else
  timeout 900 python -m pytest tests/test_k1_gpu.py tests/test_model_gpu.py -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
timeout 300 python tools/smoke_run.py 200 > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
if [ "$MODE" = "full" ]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 6000 --csv --log-file $OUT/launches_$TAG.csv \
    python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/launches_$TAG.log 2>&1
  timeout 300 python tools/gemm_bench.py > $OUT/gemm_bench_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none -k 'regex:gemm_tc' -s 2000 -c 4 -o $OUT/gemm_$TAG \
    python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/ncu_gemm_$TAG.log 2>&1
fi
SPEX_ATTN_LOG=$OUT/k1_bytes_$TAG.txt timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:tree_attn_(decode|chunk|bulk)' -s 400 -c 3 -o $OUT/k1_$TAG \
  python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/ncu_k1_$TAG.log 2>&1
echo done
