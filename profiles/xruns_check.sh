# the cross-run kernel: its GPU tests, the config-4 run-kernel time with it and without (CPHIFI_XRUNS=0),
# and an ncu source-level capture of one launch
python -m pytest tests/test_gpu_xruns.py tests/test_gpu_runs.py tests/test_gpu_dense_rows.py -x -q > gpurun_out/xr_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/xr_tests.log
VARS="0" bash profiles/runs_var_sweep.sh > gpurun_out/xr_sweep.log 2>&1
CPHIFI_XRUNS=0 VARS="0" bash profiles/runs_var_sweep.sh >> gpurun_out/xr_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xruns_kernel -c 1 -o gpurun_out/prof_xruns4 -f \
    python profiles/prof_stream.py --config 4 --iters 1 > gpurun_out/ncu_xruns4.log 2>&1
ncu -i gpurun_out/prof_xruns4.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/xruns4_src.csv 2>&1
ncu -i gpurun_out/prof_xruns4.ncu-rep --page raw --csv > gpurun_out/xruns4_raw.csv 2>&1
