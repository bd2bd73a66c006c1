timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 120 python scripts/pass_ab.py 1,8,16 2048
timeout -s KILL 120 python scripts/pass_ab.py 1,8,16 128
