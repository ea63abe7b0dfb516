for v in "" "CPHIFI_PCG_STEP_COOP=0" "CPHIFI_PCG_FUSED=0"; do echo "== $v"; env $v timeout 300 python profiles/prof_pcg_launches.py --config 4 2>&1 | tail -3; done
