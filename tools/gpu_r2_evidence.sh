# final-evidence capture: bench line, launch list of one bench step, ncu --set full of the sweep kernel
set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched --no-configs --no-fp64 > gpurun_out/ev_plain.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched --no-configs --no-fp64 > gpurun_out/ev_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout -s KILL 300 python tools/prof_tl.py 18 2 > gpurun_out/ev_prof_plain.log 2>&1 && \
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/ev_sweep_full python tools/prof_tl.py 18 2 > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ev_ncu_full.log
