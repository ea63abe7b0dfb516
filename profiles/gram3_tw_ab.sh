# register-fragment build over parts at config 4: single-warp teams (8 warps, 255 registers) vs 4-warp teams
CPHIFI_GRAM_TIMING=1 python profiles/prof_gram_parts.py config4 "1" > gpurun_out/gram_tw1.log 2>&1
CPHIFI_GRAM3_TW=4 CPHIFI_GRAM_TIMING=1 python profiles/prof_gram_parts.py config4 "1" > gpurun_out/gram_tw4.log 2>&1
python -m pytest tests/test_gpu_dense_rows.py tests/test_gpu_gram.py tests/test_gpu_full_pcg.py -x -q > gpurun_out/gram_tw_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gram_tw_tests.log
