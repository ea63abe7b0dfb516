# fresh-factor config-4 solve, row-Gram build over parts (default) vs k_gram.cu's batched build
CPHIFI_SOLVE_TIMING=1 CPHIFI_GRAM_TIMING=1 python profiles/prof_fresh_solve.py > gpurun_out/fresh_parts.log 2>&1
CPHIFI_GRAM3_PARTS=0 CPHIFI_SOLVE_TIMING=1 CPHIFI_GRAM_TIMING=1 python profiles/prof_fresh_solve.py > gpurun_out/fresh_batched.log 2>&1
