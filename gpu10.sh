cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python profiles/prof_stream.py --config 4 --iters 2 > gpurun_out/plain_p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 4 -c 2 -o gpurun_out/prof_runs_config4 python profiles/prof_stream.py --config 4 --iters 2 > gpurun_out/ncu_p.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_p.log
