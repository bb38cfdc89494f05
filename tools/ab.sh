python tools/time_eval.py 5:8388608 4 2>&1 | tail -2
