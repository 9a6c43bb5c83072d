set -o pipefail
timeout -s KILL 300 python tools/prof_posref.py 18 3 2>&1 | tail -3
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2o_posref_launches.csv python tools/prof_posref.py 18 2 > gpurun_out/r2o_ncu.log 2>&1; echo "rc=$?"
python tools/launch_table.py gpurun_out/r2o_posref_launches.csv 2>&1 | head -20
