set -o pipefail
for rep in 1 2; do
TAG=cur timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
for v in red spin; do TAG=$v PTY_LIB=variants/lib_$v.so timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1; done
done
