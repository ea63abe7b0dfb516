# B through the run kernel over the q-pass plan's parts: GPU tests and the config-4 fresh-factor solve
python -m pytest tests -m gpu -x -q > gpurun_out/rhs_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rhs_tests.log
CPHIFI_SOLVE_TIMING=1 python profiles/prof_fresh_solve.py > gpurun_out/fresh_rhs.log 2>&1
CPHIFI_RHS_PARTS=0 CPHIFI_SOLVE_TIMING=1 python profiles/prof_fresh_solve.py > gpurun_out/fresh_rhs0.log 2>&1
