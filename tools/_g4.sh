ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/g4_gu_mid python tools/gemm_one.py --model mid_policy --op gate_up --cg 2 --bn 256 --reps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/g4_lm_mid python tools/gemm_one.py --model mid_policy --op lm_head --cg 2 --bn 256 --reps 3 > /dev/null 2>&1
ls gpurun_out/g4*
