PTY_BATCH_CHUNK=400 timeout -s KILL 300 python tools/prof_batched.py 20 400 2 > gpurun_out/pb3_plain.log 2>&1 && \
PTY_BATCH_CHUNK=400 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"bk_cols_mod|bk_rows_inv|bk_rows_fwd" -s 3 -c 3 -o gpurun_out/prof_bk python tools/prof_batched.py 20 400 2 > gpurun_out/pb3_ncu.log 2>&1; echo rc=$?
