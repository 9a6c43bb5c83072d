# batched chunk-size sweep (config 5) + replica R sweep timeline
set -o pipefail
mkdir -p gpurun_out
for c in 1600 400 200 100 64 48 32; do
  echo "== chunk $c"
  PTY_BATCH_CHUNK=$c timeout -s KILL 300 python tools/prof_batched.py 80 1600 3 2>&1 | tail -1
done > gpurun_out/r2c_chunks.log 2>&1
cat gpurun_out/r2c_chunks.log
for r in 2 9 18; do
  echo "== R $r"
  PTY_TIMELINE=40 timeout -s KILL 300 python tools/prof_sweep.py $r 3 --timeline 2>&1 | tail -12
done > gpurun_out/r2c_timeline.log 2>&1
cat gpurun_out/r2c_timeline.log
