set -x
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/g2_gu8b python tools/gemm_one.py --model llama3_8b --op gate_up --cg 2 --bn 256 --reps 3 > gpurun_out/g2_ncu1.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/g2_omid python tools/gemm_one.py --model mid_policy --op o --cg 1 --bn 128 --reps 3 > gpurun_out/g2_ncu2.txt 2>&1
ls -la gpurun_out
