export PTY_SWEEP_TILES_MAX=0 PTY_CLUSTER=16
timeout -s KILL 300 python tools/prof_sweep.py 1 2 > gpurun_out/plain_c1.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_c1 python tools/prof_sweep.py 1 2 > gpurun_out/ncu_c1.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_c1.ncu-rep --page source --csv --print-source=cuda > gpurun_out/prof_c1_src.csv 2>/dev/null; echo done
