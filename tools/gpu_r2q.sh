set -o pipefail
timeout -s KILL 300 python tools/prof_posref.py 18 3 2>&1 | tail -2
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fields_registration.py tests/test_gpu_visit_api.py tests/test_gpu_acceptance.py tests/test_gpu_bench_parity.py -q -x --timeout 600 > gpurun_out/r2q_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r2q_tests.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2q_posref_launches.csv python tools/prof_posref.py 18 2 > gpurun_out/r2q_ncu.log 2>&1; echo "rc=$?"
python tools/launch_table.py gpurun_out/r2q_posref_launches.csv 2>/dev/null | head -9
