# final evidence of round 2: GPU tests, bench line + reference arm, smoke, launch list of the bench step,
# ncu --set full of the sweep kernel
set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/ev2_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/ev2_tests.log
timeout -s KILL 1200 python bench.py > gpurun_out/ev2_bench.json 2> gpurun_out/ev2_bench.err; echo "bench rc=$?"
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev2_bench_ref.json 2> gpurun_out/ev2_bench_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-single --no-batched --no-configs --no-fp64 > gpurun_out/ev2_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout -s KILL 300 python tools/prof_tl.py 18 2 > gpurun_out/ev2_prof_plain.log 2>&1 && \
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/ev2_sweep_full python tools/prof_tl.py 18 2 > gpurun_out/ev2_ncu_full.log 2>&1; echo "ncu full rc=$?"
