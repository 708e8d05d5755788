#!/bin/bash
# gpurun -- bash tools/gpu_c5_gemm.sh TAG: full ncu captures of the tcgen05 GEMMs in the config-5 (Llama-3-8B + 1.5B PRM) forward
TAG=${1:-x}; OUT=gpurun_out; mkdir -p $OUT
timeout 1500 ncu --set full --clock-control none -k 'regex:gemm_tc' -s 3000 -c 6 -o $OUT/gemm_c5_$TAG \
  python tools/model_timing.py c5_rebase_w32_q64 llama3_8b prm_1p5b > $OUT/ncu_gemm_c5_$TAG.log 2>&1
echo "ncu rc=$?"
