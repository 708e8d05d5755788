timeout -s KILL 600 python -m pytest tests/test_gemm_tc_gpu.py -x -q > gpurun_out/g5_gemm_test.txt 2>&1; echo rc=$? >> gpurun_out/g5_gemm_test.txt
tail -3 gpurun_out/g5_gemm_test.txt
timeout -s KILL 600 python tools/gemm_bench.py --sweep > gpurun_out/g5_gemm_bench.jsonl 2>&1; echo rc=$?
timeout -s KILL 300 python -m pytest tests/test_dropin_gpu.py -x -q > gpurun_out/g5_dropin.txt 2>&1; tail -3 gpurun_out/g5_dropin.txt
