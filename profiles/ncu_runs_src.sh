# Source-level ncu capture of the run kernel at config 4 (one operator launch: the first 4 are the RHS B over the parts) plus a plain timing run
set -x
python profiles/prof_stream.py --config 4 --iters 10 > gpurun_out/ps4.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 4 -c 1 -o gpurun_out/prof_runs4 -f \
    python profiles/prof_stream.py --config 4 --iters 1 > gpurun_out/ncu_runs4.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_runs4.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/runs4_src.csv 2>&1
ncu -i gpurun_out/prof_runs4.ncu-rep --page raw --csv > gpurun_out/runs4_raw.csv 2>&1
