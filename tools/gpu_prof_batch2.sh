timeout -s KILL 300 python tools/prof_batched.py 80 1600 2 > gpurun_out/pb_plain.log 2>&1; cat gpurun_out/pb_plain.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pb_launches.csv python tools/prof_batched.py 80 1600 1 > gpurun_out/pb_ncu.log 2>&1; echo "rc=$?"
