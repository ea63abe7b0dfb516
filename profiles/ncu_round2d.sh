# ncu evidence of the new default run kernel (RV_FOLDZ loop): launch list of the bench command and one
# --set full capture of the operator's run kernel (the first 4 run-kernel launches are the right-hand side B)
set -x
C="python bench.py --steps 20 --warmup 3 --secondary 0 --cpu-seconds 1"
$C > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_l.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 4 -c 1 -o gpurun_out/prof_runs_r2d -f $C > gpurun_out/ncu_f.log 2>&1; echo "ncu2 rc=$?"
python profiles/ncu_summary.py full gpurun_out/prof_runs_r2d.ncu-rep gpurun_out/ncu_full_runs_config4.json; echo "sum rc=$?"
python profiles/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_config4.txt
