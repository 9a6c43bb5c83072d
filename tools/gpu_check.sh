set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout -s KILL 240 python __graft_entry__.py --smoke 2>&1 | tail -20
timeout -s KILL 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -30
