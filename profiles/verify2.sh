timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
CPHIFI_DEBUG=1 timeout 600 python profiles/prof_solves.py 2>&1 | tail -20
