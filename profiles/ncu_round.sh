# ncu evidence for profiles/: launch list of the bench command, full captures of the top kernels
C="python bench.py --steps 20 --warmup 3 --secondary 0 --cpu-seconds 1"
$C > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fused_matvec -s 5 -c 1 -o gpurun_out/prof_fused $C > gpurun_out/ncu_f.log 2>&1; echo "ncu fused rc=$?"
python profiles/prof_aligned2.py config2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mttkrp_v3|sandwich2" -s 3 -c 3 -o gpurun_out/prof_aligned python profiles/prof_aligned2.py config2 > gpurun_out/ncu_a.log 2>&1; echo "ncu aligned rc=$?"
