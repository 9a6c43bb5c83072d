# Full refresh: GPU tests, bench line, reference arm, launch list, one ncu --set full capture.
set -o pipefail
R=${R:-18}
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched --no-configs > gpurun_out/plain_bench.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched --no-configs > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
PTY_SWEEP_TILES_MAX=0 timeout -s KILL 300 python tools/prof_sweep.py $R 2 > gpurun_out/plain_prof.log 2>&1 && \
PTY_SWEEP_TILES_MAX=0 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_full python tools/prof_sweep.py $R 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
