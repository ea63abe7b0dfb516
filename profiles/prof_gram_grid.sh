# Row-Gram build device time vs the build's CTAs per SM (partition granularity); "auto" = the library's choice
for c in auto 4 8; do echo "== CTAs/SM $c"; if [ $c = auto ]; then E=""; else E="CPHIFI_GRAM_CTAS_PER_SM=$c"; fi
env $E CPHIFI_GRAM_TIMING=1 python profiles/prof_gram_build.py config3 config4 2>&1 | grep -E "gram build" | sed -n '2p;4p'; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
