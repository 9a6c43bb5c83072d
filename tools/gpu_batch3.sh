for G in 48 56 64 128 200; do echo "G=$G"; PTY_K4_GROUPS=$G timeout -s KILL 300 python tools/prof_batched.py 20 400 4; done
timeout -s KILL 300 python tools/prof_batched.py 20 400,400 4
