# config 4 PCG: graph vs host-loop solve times under library switches
for v in "" "CPHIFI_GEMM_TMA=0" "CPHIFI_PCG_FUSED=0"; do
echo "== $v"; env $v python profiles/prof_pcg_launches.py --config 4 --ab 5 2>&1 | awk '/graph=1/{if(n>0)a+=$5;n++} /graph=0/{b+=$5;m++} END{print "graph", a/(n-1), "host", b/m}'
done
