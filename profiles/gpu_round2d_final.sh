# round-2 evidence at HEAD (balanced shards, row-sharded operator, plan-column slack): GPU suite twice
# (flakiness check), smoke, bench line, reference arm, launch list of the bench command
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest(2) rc=$?"
tail -1 gpurun_out/pytest_gpu2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
C="python bench.py --steps 20 --warmup 3 --secondary 0 --cpu-seconds 1"
$C > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_l.log 2>&1; echo "ncu1 rc=$?"
