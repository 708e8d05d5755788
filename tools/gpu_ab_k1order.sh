#!/bin/bash
# gpurun -- bash tools/gpu_ab_k1order.sh TAG: alternating A/B of the K1 claim order on config 2 (mid shapes)
TAG=${1:-x}; OUT=gpurun_out; mkdir -p $OUT
python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > /dev/null 2>&1  # warm
for i in 1 2 3; do
  for v in 1 0; do
    SPEX_K1_QLPT=$v python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('QLPT=$v', 'step_ms', round(d['step_ms'],1), 'k1_ms', round(d['attn_ms'],1), 'k1_TBs', round(d['attn_alg_bytes']/(d['attn_ms']/1e3)/1e12,3))"
  done
done | tee $OUT/ab_k1order_$TAG.txt
