set -o pipefail
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.json
tail -3 gpurun_out/bench_full.err
