timeout 600 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -1
python profiles/prof_pcg_launches.py --config 4 --ab 4 2>&1 | tail -8
ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg4.csv python profiles/prof_pcg_launches.py --config 4 > /dev/null 2>&1; echo ncu=$?
