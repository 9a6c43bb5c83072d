#!/bin/bash
# A/B of variant libraries (variants/lib_<name>.so) against the default build:
# 18-replica sweep time, interleaved, plus the benchmarked-config parity test per variant.
# usage: tools/gpu_r2x.sh name1 name2 ...
mkdir -p gpurun_out
for v in "$@"; do
  PTY_LIB=variants/lib_$v.so timeout 300 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "18_replicas or w512" 2>&1 | tail -1 | sed "s/^/parity $v: /"
done
for i in 1 2; do
  TAG=default timeout 120 python tools/ab_time.py 18 8 2>&1 | grep R=
  for v in "$@"; do PTY_LIB=variants/lib_$v.so TAG=$v timeout 120 python tools/ab_time.py 18 8 2>&1 | grep R=; done
done
