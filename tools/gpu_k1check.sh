#!/bin/bash
# gpurun -- bash tools/gpu_k1check.sh TAG: K1 correctness tests + config-5 timing (A/B of the GQA K1 kernel)
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_k1_gpu.py tests/test_model_gpu.py -q -x --timeout 600 > $OUT/k1check_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/k1check_$TAG.log
tail -3 $OUT/k1check_$TAG.log
for i in 1 2; do timeout 600 python tools/model_timing.py c5_rebase_w32_q64 llama3_8b prm_1p5b > $OUT/c5_timing_${TAG}_$i.json 2>&1; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/c5_timing_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "step_ms", round(d["step_ms"],1), "attn_ms", round(d["attn_ms"],1), "k1 TB/s", round(d["attn_alg_bytes"]/(d["attn_ms"]/1e3)/1e12,3))
    except Exception as e: print(f, e)
PY
