set -x
export PTY_SWEEP_TILES_MAX=0
PTY_CLUSTER=0 PTY_TIMELINE=12 timeout 120 python tools/prof_sweep.py 16 2 --timeline
PTY_CLUSTER=16 PTY_TIMELINE=12 timeout 120 python tools/prof_sweep.py 1 2 --timeline
PTY_CLUSTER=16 PTY_TIMELINE=12 timeout 120 python tools/prof_sweep.py 8 2 --timeline
