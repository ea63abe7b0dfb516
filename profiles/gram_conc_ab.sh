# row-Gram build at config 4: dense rows' parts concurrent on the plan's second stream (default) vs sequential
timeout 600 python -m pytest tests/test_gpu_dense_rows.py tests/test_gpu_gram.py -x -q -m gpu > gpurun_out/gram_conc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gram_conc_tests.log
for c in 1 0 1 0; do CPHIFI_GRAM_CONCURRENT=$c timeout 300 python profiles/prof_gram_parts.py config4 "1" > gpurun_out/gram_conc_$c.log 2>&1; echo "conc=$c rc=$?"; tail -2 gpurun_out/gram_conc_$c.log; done
