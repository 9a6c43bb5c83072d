timeout -s KILL 600 python -m pytest tests/test_gpu_batched.py -q --timeout 300 2>&1 | tail -2
timeout -s KILL 300 python tools/prof_batched.py 20 400 2 > gpurun_out/pb_plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/pb_launches.csv python tools/prof_batched.py 20 400 2 > gpurun_out/pb_ncu.log 2>&1
echo rc=$?
