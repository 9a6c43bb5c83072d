set -o pipefail
timeout -s KILL 600 python tools/overlap_test.py 2>&1 | tail -4
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x --timeout 600 > gpurun_out/r2n_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r2n_tests.log
timeout -s KILL 900 python bench.py --steps 6 --warmup 3 --no-cpu --no-batched --no-configs --no-fp64 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2n_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e'])"
