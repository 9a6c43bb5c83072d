timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3
for R in 1 4 8 16; do timeout -s KILL 300 python tools/prof_sweep.py $R 4 | tail -1; done
for R in 4 8; do PTY_SWEEP_TILES_MAX=0 timeout -s KILL 300 python tools/prof_sweep.py $R 4 | tail -1; done
PTY_SWEEP_TILES_MAX=0 timeout -s KILL 300 python tools/prof_sweep.py 24 4 | tail -1
