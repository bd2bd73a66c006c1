timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 120 python scripts/pass_timeline.py 8 128 2>&1 | grep -v cta | tail -12
timeout -s KILL 120 python scripts/pass_ab.py 1,8,32 128
DD_PASS_PREFETCH=0 timeout -s KILL 120 python scripts/pass_ab.py 8 128
