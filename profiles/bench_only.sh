# the default bench line (config 4 headline + secondary numbers)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
