# ncu --set full of the fused PCG vector step and of the eigenbasis GEMM (config 4, host-loop solve)
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:pcg_step_fused -s 3 -c 1 -o gpurun_out/prof_step python profiles/prof_pcg_launches.py --config 4 > gpurun_out/ncu_step.log 2>&1; echo "ncu1 rc=$?"
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:mttkrp_v3 -s 4 -c 2 -o gpurun_out/prof_gemm4 python profiles/prof_pcg_launches.py --config 4 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu2 rc=$?"
