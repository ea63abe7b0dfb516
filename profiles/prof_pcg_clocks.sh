# config 4 PCG: graph vs host-loop solves with SM clock / power / throttle sampling alongside
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/clk.csv &
SMI=$!
python profiles/prof_pcg_launches.py --config 4 --ab 60 > gpurun_out/ab4.log 2>&1
kill $SMI
grep -c "graph=1" gpurun_out/ab4.log; awk '/graph=1/{a+=$5;n++} /graph=0/{b+=$5;m++} END{print "graph", a/n, "host", b/m}' gpurun_out/ab4.log
