# config-2 aligned solve after the Gram fork and the split-reduce load batching; launch list; tests
python profiles/prof_aligned2.py > gpurun_out/al2b.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/al2b_launches.csv python profiles/prof_aligned2.py > gpurun_out/al2b_ncu.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_aligned_baselines.py tests/test_gpu_als.py -x -q > gpurun_out/al2b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/al2b_tests.log
