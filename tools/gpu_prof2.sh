timeout -s KILL 300 python tools/prof_sweep.py 16 2 > gpurun_out/plain16.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_r16 python tools/prof_sweep.py 16 2 > gpurun_out/ncu_r16.log 2>&1
tail -2 gpurun_out/ncu_r16.log
