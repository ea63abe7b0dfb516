# launch list of the config-2 aligned solve (MTTKRP, Gram, decoupled sandwich) and an ncu --set full of the sandwich
python profiles/prof_aligned2.py > gpurun_out/al2.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/al2_launches.csv python profiles/prof_aligned2.py > gpurun_out/al2_ncu.log 2>&1; echo "ncu rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sandwich3 -s 4 -c 2 -o gpurun_out/prof_sand3 -f python profiles/prof_aligned2.py > gpurun_out/al2_ncu2.log 2>&1; echo "ncu2 rc=$?"
ncu -i gpurun_out/prof_sand3.ncu-rep --page raw --csv > gpurun_out/sand3_raw.csv 2>&1
