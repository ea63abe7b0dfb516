# run-kernel inner-loop variants (CPHIFI_RUNS_VAR, k_runs.cu RV_* bits) at config 4, one process each
for v in ${VARS:-0 1 2 3 4 7 20 23 28 31}; do
  CPHIFI_RUNS_VAR=$v python profiles/prof_stream.py --config ${CONFIG:-4} --iters 10 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['variants'][0]; print('var $v', round(d['stream_ms'],3), round(d['app_ms'],3), repr(d['y_sum']), repr(d['y_norm']))"
done
