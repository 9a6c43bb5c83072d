set -o pipefail
for rep in 1 2; do
TAG=r2a bash -c 'cd variants/r2a && timeout -s KILL 300 python tools/ab_time.py 18 8' 2>&1 | tail -1
TAG=cur timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
TAG=cur_pair PTY_SLOT_PAIR=1 timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
TAG=regstage PTY_LIB=variants/lib_regstage.so timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
done
