#!/bin/bash
# gpurun -- bash tools/gpu_ab_lib.sh TAG: same-box A/B of the built library against
# paper_2605_10195_b200/lib/ab/libspex_b200_base.so (SPEX_LIB_PATH), alternating
# runs of config 5 (8B + 1.5B PRM) and config 2 (mid) timing; K1 tests first.
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_k1_gpu.py tests/test_model_gpu.py tests/test_gemm_tc_gpu.py -q -x --timeout 600 > $OUT/ab_tests_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/ab_tests_$TAG.log
tail -2 $OUT/ab_tests_$TAG.log
BASE=paper_2605_10195_b200/lib/ab/libspex_b200_base.so
NEW=paper_2605_10195_b200/lib/libspex_b200.so
for i in 1 2; do
  for v in base new; do
    L=$BASE; [ $v = new ] && L=$NEW
    SPEX_LIB_PATH=$L timeout 600 python tools/model_timing.py c5_rebase_w32_q64 llama3_8b prm_1p5b > $OUT/ab_${TAG}_c5_${v}_$i.json 2>&1
    SPEX_LIB_PATH=$L timeout 600 python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/ab_${TAG}_c2_${v}_$i.json 2>&1
  done
done
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/ab_${TAG}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "step_ms", round(d["step_ms"],1), "attn_ms", round(d["attn_ms"],1), "k1 TB/s", round(d["attn_alg_bytes"]/(d["attn_ms"]/1e3)/1e12,3))
    except Exception as e: print(f, e)
PY
