# v5 (cluster-multicast sandwich): variant tests, then config-2 decoupled timing v3 vs v5
timeout 300 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "sandwich" > gpurun_out/v5_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/v5_tests.log
for v in 0 8 4 2; do CPHIFI_SANDWICH_V5=$v timeout 120 python profiles/prof_aligned2.py > gpurun_out/al2_v5_$v.log 2>&1; echo "v5=$v rc=$?"; tail -1 gpurun_out/al2_v5_$v.log; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/al2_launches_v5.csv python profiles/prof_aligned2.py > /dev/null 2>&1; echo "ncu rc=$?"
