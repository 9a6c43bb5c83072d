PTY_SWEEP_TILES_MAX=0 PTY_TIMELINE=120 timeout -s KILL 300 python tools/tl_cta.py 18 2 2>&1 | tail -14
