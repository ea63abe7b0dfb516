# ncu (full, source) of the register-fragment row-Gram build over a factor-block part at config 4
# (CPHIFI_GRAM3_PARTS=1, the third launch: a dense-rows part)
ncu --set full --clock-control none --import-source on -k regex:gram3_kernel -s 2 -c 1 -o gpurun_out/prof_gram3p -f \
    python profiles/prof_gram_parts.py config4 "1" > gpurun_out/ncu_gram3p.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_gram3p.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/gram3p_src.csv 2>&1
ncu -i gpurun_out/prof_gram3p.ncu-rep --page raw --csv > gpurun_out/gram3p_raw.csv 2>&1
