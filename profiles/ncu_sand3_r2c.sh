# ncu --set full of the config-2 decoupled chain: reduce_splits, to_rows_padded, sandwich3 (both phases)
ncu --set full --clock-control none --import-source on -k regex:"sandwich3|reduce_splits|to_rows_padded" -s 8 -c 4 -o gpurun_out/prof_sand3 -f python profiles/prof_aligned2.py > gpurun_out/al2_ncu2.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_sand3.ncu-rep --page raw --csv > gpurun_out/sand3_raw.csv 2>&1
ncu -i gpurun_out/prof_sand3.ncu-rep --page details --csv > gpurun_out/sand3_details.csv 2>&1
