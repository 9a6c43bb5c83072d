set -o pipefail
for rep in 1 2; do
TAG=r2a bash -c 'cd variants/r2a && timeout -s KILL 300 python tools/ab_time.py 18 8' 2>&1 | tail -1
TAG=cur timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
for v in ch8 ch2; do
TAG=$v PTY_LIB=variants/lib_$v.so timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
done
done
