#!/bin/bash
# gpurun -- bash tools/gpu_sel.sh TAG pytest-args...: selected GPU tests only (no bench).
TAG=${1:-x}; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest "$@" -q -rf --timeout 600 > $OUT/pytest_sel_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sel_$TAG.log
tail -40 $OUT/pytest_sel_$TAG.log
