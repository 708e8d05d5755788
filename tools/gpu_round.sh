#!/bin/bash
# One gpurun call: GPU tests, smoke, bench line (+ reference arm), ncu launch list,
# full ncu captures of K1 and of the projection GEMMs, config-4 probe and control
# phases. Usage: gpurun -- bash tools/gpu_round.sh TAG [quick]
TAG=${1:-r02}
MODE=${2:-full}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
if [ "$MODE" = "full" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
if [ "$MODE" = "full" ]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 6000 --csv --log-file $OUT/launches_$TAG.csv \
    python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/launches_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:gemm_tc' -s 2000 -c 4 -o $OUT/gemm_$TAG \
    python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/ncu_gemm_$TAG.log 2>&1
  timeout 600 python tools/c4_probe.py > $OUT/c4_probe_$TAG.jsonl 2>&1
  timeout 300 python tools/ctl_phases.py c4_rest_w4_q4096 c2_rebase_w16_q256 c3_rstar_w4_q512 > $OUT/ctl_phases_$TAG.txt 2>&1
fi
SPEX_ATTN_LOG=$OUT/k1_bytes_$TAG.txt timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:tree_attn_(decode|bulk)' -s 400 -c 3 -o $OUT/k1_$TAG \
  python tools/model_timing.py c2_rebase_w16_q256 mid_policy mid_prm > $OUT/ncu_k1_$TAG.log 2>&1
echo done
