set -o pipefail
mkdir -p gpurun_out
PTY_SWEEP_TILES_MAX=0 timeout -s KILL 300 python tools/prof_tl.py 2 2 > gpurun_out/r2e_plain.log 2>&1 && \
PTY_SWEEP_TILES_MAX=0 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/r2e_r2 python tools/prof_tl.py 2 2 > gpurun_out/r2e_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2e_ncu.log
