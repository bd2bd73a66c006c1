timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 120 python scripts/pass_ab.py 1,8,16 128
DD_PASS_BALANCE=0 timeout -s KILL 120 python scripts/pass_ab.py 1,8,16 128
timeout -s KILL 120 python scripts/sm_speed.py 2>&1 | head -3
DD_PASS_BALANCE=0 timeout -s KILL 120 python scripts/sm_speed.py 2>&1 | head -3
