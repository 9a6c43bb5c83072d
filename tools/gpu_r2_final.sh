set -o pipefail
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/fin_tests.log
timeout -s KILL 1200 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/fin_bench.json
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err; echo "ref rc=$?"
tail -c 400 gpurun_out/fin_bench_ref.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
