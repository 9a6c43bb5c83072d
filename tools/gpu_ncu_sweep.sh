# ncu --set full of the sweep kernel (18 own-dataset replicas), source page included
mkdir -p gpurun_out
timeout -s KILL 300 python tools/prof_tl.py 18 2 > gpurun_out/ncu_plain.log 2>&1 && \
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_full python tools/prof_tl.py 18 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
