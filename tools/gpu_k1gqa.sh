#!/bin/bash
# gpurun -- bash tools/gpu_k1gqa.sh TAG: source-level ncu of the GQA K1 kernel (config 5, Llama-3-8B shape)
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
SPEX_ATTN_LOG=$OUT/k1gqa_bytes_$TAG.txt timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:tree_attn_wmma -s 300 -c 2 -o $OUT/k1gqa_$TAG python tools/model_timing.py c5_rebase_w32_q64 llama3_8b prm_1p5b \
  > $OUT/ncu_k1gqa_$TAG.log 2>&1
echo "ncu rc=$?"
timeout 600 python tools/model_timing.py c5_rebase_w32_q64 llama3_8b prm_1p5b > $OUT/c5_timing_$TAG.json 2>&1
cat $OUT/c5_timing_$TAG.json | tail -2
