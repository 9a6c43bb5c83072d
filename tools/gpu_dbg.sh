export PTY_SWEEP_TILES_MAX=0 PTY_CLUSTER=0 PTY_TIMELINE=12
for d in ${DBGS:-0 4 8 16 28}; do echo "debug=$d"; PTY_DEBUG=$d timeout 120 python tools/prof_sweep.py 16 2 --timeline 2>&1 | sed -n 4,6p; done
