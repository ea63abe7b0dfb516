# config-1 fused operator: partition / CTAs-per-SM variants (device time per application)
for v in "" "CPHIFI_FUSED_OCC=1" "CPHIFI_FUSED_OCC=1 CPHIFI_EQUAL_PART=148" "CPHIFI_EQUAL_PART=296" "CPHIFI_EQUAL_PART=148" "CPHIFI_EQUAL_PART=200"; do
  echo "== $v"; env $v python profiles/prof_matvec.py --iters 30 2>&1 | grep -E "flush|exit|barrier|B done|B loop"
done
ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg4w.csv python profiles/prof_pcg_launches.py --config 4 > gpurun_out/pcg4w_ncu.log 2>&1; echo "ncu rc=$?"
