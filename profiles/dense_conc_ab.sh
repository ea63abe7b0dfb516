# dense rows concurrent with the run kernel's parts (second stream; issued before part 0 / after part 0)
for f in 0 1; do
  CPHIFI_DENSE_FORK_AT=$f python bench.py --steps 30 --warmup 3 --secondary 0 --cpu-seconds 1 > gpurun_out/conc_f$f.json 2>&1
done
CPHIFI_DENSE_CONCURRENT=0 python bench.py --steps 30 --warmup 3 --secondary 0 --cpu-seconds 1 > gpurun_out/conc0.json 2>&1
