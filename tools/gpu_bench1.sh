set -x
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -15
for R in 1 4 8 16; do
  timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --replicas $R --no-cpu --no-single 2>&1 | tail -3
done
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 2>&1 | tail -3
