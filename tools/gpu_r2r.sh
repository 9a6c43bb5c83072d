set -o pipefail
timeout -s KILL 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_batched.py -q -x --timeout 600 2>&1 | tail -2
for rep in 1 2; do
echo "== default"; timeout -s KILL 300 python tools/prof_batched.py 80 1600 3 2>&1 | tail -1
for v in bk6 bk4; do echo "== $v"; PTY_LIB=variants/lib_$v.so timeout -s KILL 300 python tools/prof_batched.py 80 1600 3 2>&1 | tail -1; done
done
