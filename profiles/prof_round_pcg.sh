# GPU tests + per-iteration kernel breakdown of the config 3 / 4 PCG solves (host-driven loop under ncu, warm caches)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in 4 3; do
python profiles/prof_pcg_launches.py --config $c 2>&1 | tail -3
CPHIFI_PCG_FUSED=0 python profiles/prof_pcg_launches.py --config $c 2>&1 | tail -2
ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg$c.csv python profiles/prof_pcg_launches.py --config $c > gpurun_out/pcg${c}_ncu.log 2>&1; echo "ncu$c rc=$?"
done
