# round 2 first pass: GPU tests (PARITY lines), bench line, timeline of the sweep
set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -s --timeout 600 > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2a_tests.log; grep PARITY gpurun_out/r2a_tests.log
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2a_bench.json
