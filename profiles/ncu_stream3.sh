# ncu --set full of the k_stream.cu operator launch at config 3 (q = 2e7 sample, same per-observation work)
C="python profiles/prof_large.py --config 3 --q 200000000 --trace 0 --iters 2"
$C > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 1 -o gpurun_out/prof_stream3 -f $C > gpurun_out/ncu3.log 2>&1; echo rc=$?
