timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 1 0; do echo "== CPHIFI_HOST_X_FUSED=$v"; CPHIFI_HOST_X_FUSED=$v python bench.py --secondary 0 --cpu-seconds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"; done
