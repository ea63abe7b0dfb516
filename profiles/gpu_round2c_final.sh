# round-2 evidence at HEAD (fresh container re-entry): GPU suite, smoke, bench line, reference arm, launch list of the bench
# command, ncu --set full of the headline's dominant kernel (the operator's run kernel: the first 4
# run-kernel launches are the right-hand side B over the parts)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
C="python bench.py --steps 20 --warmup 3 --secondary 0 --cpu-seconds 1"
$C > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_l.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 4 -c 1 -o gpurun_out/prof_runs_r2c -f $C > gpurun_out/ncu_f.log 2>&1; echo "ncu2 rc=$?"
ncu -i gpurun_out/prof_runs_r2c.ncu-rep --page raw --csv > gpurun_out/runs_r2c_raw.csv 2>&1
ncu --set full --clock-control none -k regex:dense_rows_kernel -s 3 -c 1 -o gpurun_out/prof_dense_r2c -f $C > gpurun_out/ncu_d.log 2>&1; echo "ncu3 rc=$?"
ncu -i gpurun_out/prof_dense_r2c.ncu-rep --page raw --csv > gpurun_out/dense_r2c_raw.csv 2>&1
