set -o pipefail
timeout -s KILL 900 python -m pytest tests/test_gpu_cli.py -q -x --timeout 600 2>&1 | tail -15
