timeout 600 python tools/dp_leg_check.py 2>&1 | tail -3
