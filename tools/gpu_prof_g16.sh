export PTY_SWEEP_TILES_MAX=0 PTY_CLUSTER=${PTY_CLUSTER:-0}
R=${R:-16}
timeout -s KILL 300 python tools/prof_sweep.py $R 2 > gpurun_out/plain_g.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_g python tools/prof_sweep.py $R 2 > gpurun_out/ncu_g.log 2>&1; echo "ncu rc=$?"
