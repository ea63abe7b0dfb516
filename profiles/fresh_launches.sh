# launch list of the config-4 fresh-factor solves (subproblem: B, V; solve: G build, PCG)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fresh_launches.csv python profiles/prof_fresh_solve.py > gpurun_out/fresh_l.log 2>&1; echo "ncu rc=$?"
