timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
timeout -s KILL 300 python tools/prof_sweep.py 1 4
timeout -s KILL 300 python tools/prof_sweep.py 4 3
timeout -s KILL 300 python tools/prof_sweep.py 16 3
