set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r2g_tests.log
PTY_SWEEP_TILES_MAX=0 PTY_TIMELINE=60 timeout -s KILL 300 python tools/tl_phases.py 18 2 2>&1 | tail -7
timeout -s KILL 900 python bench.py --steps 6 --warmup 3 --no-cpu --no-batched --no-configs --no-fp64 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2g_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'])"
