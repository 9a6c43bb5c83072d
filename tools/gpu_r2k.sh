set -o pipefail
bash tools/gpu_r2j.sh
timeout -s KILL 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_batched.py tests/test_gpu_bench_parity.py -q -x --timeout 600 > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2k_tests.log
