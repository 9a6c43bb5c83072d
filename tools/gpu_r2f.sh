set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_subpixel.py -q -s -x --timeout 300 > gpurun_out/r2f_subpixel.log 2>&1; echo "subpixel rc=$?"
tail -15 gpurun_out/r2f_subpixel.log
