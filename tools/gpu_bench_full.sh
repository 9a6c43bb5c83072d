set -o pipefail
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.json
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-single > gpurun_out/plain_bench.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-single > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 300 python tools/prof_sweep.py 16 2 > gpurun_out/plain16.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_sweep_r16 python tools/prof_sweep.py 16 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
