timeout -s KILL 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -3
timeout -s KILL 300 python tools/prof_batched.py 20 400 3
for G in 8 32 64; do PTY_K4_GROUPS=$G timeout -s KILL 300 python tools/prof_batched.py 20 400 3; done
timeout -s KILL 400 python tools/prof_batched.py 80 1600,6400 2
timeout -s KILL 300 python tools/prof_sweep.py 16 3
