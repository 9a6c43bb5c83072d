timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -4
timeout -s KILL 300 python tools/prof_sweep.py 1 4 --barrier
timeout -s KILL 300 python tools/prof_sweep.py 16 3
timeout -s KILL 300 python tools/prof_sweep.py 1 2 > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_r1 python tools/prof_sweep.py 1 2 > gpurun_out/ncu_r1.log 2>&1
tail -3 gpurun_out/ncu_r1.log
