# ncu captures of the kernels added late in round 1: DMMA row-Gram build (config 3), stream kernel
# with the prefetch ring (config 4), batched row least squares, MTTKRP mode 1 / 2
python profiles/prof_gram.py config3 > /dev/null 2>&1
CPHIFI_GRAM_DMMA=1 ncu --set full --clock-control none -k regex:gram_build_dmma -c 1 -o gpurun_out/prof_gram3 python profiles/prof_gram.py config3 > gpurun_out/ncu_g3.log 2>&1; echo "gram rc=$?"
ncu --set full --clock-control none -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_stream4pf python profiles/prof_large.py --config 4 --coalesce 1 --trace 0 --iters 2 > gpurun_out/ncu_s4pf.log 2>&1; echo "stream rc=$?"
ncu --set full --clock-control none -k regex:"mttkrp_v3|rowls" -c 4 -o gpurun_out/prof_als python -m pytest tests/test_gpu_als.py -q -k "middle_and_last or finite_update_vs" > gpurun_out/ncu_als.log 2>&1; echo "als rc=$?"
