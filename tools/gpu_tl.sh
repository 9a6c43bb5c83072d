timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
for R in 1 16; do PTY_TIMELINE=16 timeout -s KILL 300 python tools/prof_sweep.py $R 3 --timeline; done
for R in 4 8; do timeout -s KILL 300 python tools/prof_sweep.py $R 3; done
