set -o pipefail
for rep in 1 2; do
TAG=cur timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
for v in p1cp p2pf; do
TAG=$v PTY_LIB=variants/lib_$v.so timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
done
done
timeout -s KILL 900 python bench.py --steps 6 --warmup 3 --no-cpu --no-batched --no-configs --no-fp64 > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2m_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e'])"
