# Row-Gram build v1 vs v2 at full size (device time, CUDA events) + GPU gram tests
timeout 600 python -m pytest tests/test_gpu_gram.py -x -q 2>&1 | tail -2
for v in 0 1; do echo "== CPHIFI_GRAM_V2=$v"; CPHIFI_GRAM_V2=$v CPHIFI_GRAM_TIMING=1 python profiles/prof_gram_build.py config3 config4 2>&1 | grep -E "gram build"; done
