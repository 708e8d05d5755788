set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 600 python -m pytest tests/test_gemm_tc_gpu.py -x -q > gpurun_out/g1_gemm_test.txt 2>&1; echo rc=$? >> gpurun_out/g1_gemm_test.txt
tail -5 gpurun_out/g1_gemm_test.txt
timeout -s KILL 600 python tools/gemm_bench.py --sweep > gpurun_out/g1_gemm_bench.jsonl 2>&1; echo rc=$?
timeout -s KILL 900 python -m pytest tests/test_model_gpu.py -x -q > gpurun_out/g1_model_test.txt 2>&1; echo rc=$? >> gpurun_out/g1_model_test.txt
tail -5 gpurun_out/g1_model_test.txt
