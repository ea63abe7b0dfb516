# config-2 decoupled sandwich: v3 (default) vs v4 (split-K) timings and launch lists
python profiles/prof_aligned2.py > gpurun_out/al2_v3.log 2>&1; echo "v3 rc=$?"; cat gpurun_out/al2_v3.log | tail -2
CPHIFI_SANDWICH_V4=1 python profiles/prof_aligned2.py > gpurun_out/al2_v4.log 2>&1; echo "v4 rc=$?"; cat gpurun_out/al2_v4.log | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/al2_launches_v3.csv python profiles/prof_aligned2.py > /dev/null 2>&1; echo "ncu rc=$?"
CPHIFI_SANDWICH_V4=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/al2_launches_v4.csv python profiles/prof_aligned2.py > /dev/null 2>&1; echo "ncu rc=$?"
