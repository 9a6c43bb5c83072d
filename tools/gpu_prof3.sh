timeout -s KILL 300 python tools/prof_sweep.py 16 2 > gpurun_out/plain16.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_lines_r16 python tools/prof_sweep.py 16 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched > gpurun_out/plain_bench.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
