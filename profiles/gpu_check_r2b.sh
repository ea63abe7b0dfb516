# full GPU suite, then the ncu capture of the register-fragment build over a part (config 4)
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2b.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputest_r2b.log
bash profiles/ncu_gram3_parts.sh
