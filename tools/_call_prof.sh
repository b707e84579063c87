python tools/qb_calls.py 2>&1 | tail -27
