set -o pipefail
mkdir -p gpurun_out
for r in 2 9 18; do
  echo "== R $r (lines kernel)"
  PTY_SWEEP_TILES_MAX=0 PTY_TIMELINE=60 timeout -s KILL 300 python tools/tl_phases.py $r 2 2>&1 | tail -7
done > gpurun_out/r2d_phases.log 2>&1
cat gpurun_out/r2d_phases.log
timeout -s KILL 900 python bench.py --steps 6 --warmup 3 --no-cpu --no-batched > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2d_bench.json; tail -5 gpurun_out/r2d_bench.err
