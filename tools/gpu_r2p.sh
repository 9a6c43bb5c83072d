set -o pipefail
PTY_NARROW=1 timeout -s KILL 900 python -m pytest tests/test_gpu_bench_parity.py -q -x -s -k "18_replicas and fp32" --timeout 600 2>&1 | grep -E "PARITY|passed|failed|Error" | head -5
for rep in 1 2; do
TAG=cur timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
TAG=narrow PTY_NARROW=1 timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
done
