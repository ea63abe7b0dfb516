timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python profiles/prof_pcg_launches.py --config 4 --ab 3 2>&1 | tail -3
python profiles/prof_pcg_launches.py --config 3 --ab 3 2>&1 | grep "graph=1" | tail -2
ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg4.csv python profiles/prof_pcg_launches.py --config 4 > /dev/null 2>&1; echo ncu=$?
