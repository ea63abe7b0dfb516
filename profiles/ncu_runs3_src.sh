# source-level ncu of the run kernel at config 3 (one launch) and a plain timing run
python profiles/prof_stream.py --config 3 --iters 10 > gpurun_out/ps3.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:runs_kernel -c 1 -o gpurun_out/prof_runs3 -f \
    python profiles/prof_stream.py --config 3 --iters 1 > gpurun_out/ncu_runs3.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_runs3.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/runs3_src.csv 2>&1
ncu -i gpurun_out/prof_runs3.ncu-rep --page raw --csv > gpurun_out/runs3_raw.csv 2>&1
