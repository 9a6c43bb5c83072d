for r in 2 18; do echo "== R $r"; PTY_LIB=variants/lib_probe.so PTY_SWEEP_TILES_MAX=0 timeout -s KILL 300 python tools/probe_read.py $r 2>&1 | tail -14; done
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -2
