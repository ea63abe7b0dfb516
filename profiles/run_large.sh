# GPU check of the large-plan operator: parity tests + configs 3 / 4 (raw and coalesced) timings
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 3 4; do python profiles/prof_large.py --config $c --trace 0 2>&1 | tail -1 | cut -c1-330; done
python profiles/prof_large.py --config 4 --coalesce 1 --trace 0 2>&1 | tail -1 | cut -c1-330
