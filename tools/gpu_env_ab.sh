#!/bin/bash
# A/B of environment knobs on the default library: tools/gpu_env_ab.sh "VAR=a" "VAR=b" ...
for i in 1 2; do
  TAG=default timeout 120 python tools/ab_time.py 18 6 2>&1 | grep R=
  for e in "$@"; do env $e TAG="$e" timeout 120 python tools/ab_time.py 18 6 2>&1 | grep R=; done
done
