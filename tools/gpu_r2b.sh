# visit API tests + full gpu suite quick
set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_visit_api.py -q -x --timeout 300 > gpurun_out/r2b_visit.log 2>&1; echo "visit rc=$?"
tail -15 gpurun_out/r2b_visit.log
