#!/bin/bash
# gpurun -- bash tools/gpu_bench_2rank.sh TAG: bench.py's multi-rank path (torchrun, 2 ranks) on ONE GPU
# (SPEX_BENCH_ONE_GPU=1: gloo group, both ranks on cuda:0, time-sliced): split sharding end to end.
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
for SH in split independent; do
  SPEX_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 1 --warmup 1 --control-only 0 \
    --named-shapes 0 --sharding $SH > $OUT/bench2_${TAG}_$SH.json 2> $OUT/bench2_${TAG}_$SH.err
  echo "$SH rc=$?"; tail -c 600 $OUT/bench2_${TAG}_$SH.json; tail -3 $OUT/bench2_${TAG}_$SH.err
done
