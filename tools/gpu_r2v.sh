set -o pipefail
for rep in 1 2; do
TAG=cur timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
TAG=pair PTY_SLOT_PAIR=1 timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1
for off in 1 2 3; do TAG=pair_off$off PTY_SLOT_PAIR=1 PTY_PAIR_OFFSET=$off timeout -s KILL 300 python tools/ab_time.py 18 8 2>&1 | tail -1; done
done
PTY_SLOT_PAIR=1 PTY_PAIR_OFFSET=2 PTY_SWEEP_TILES_MAX=0 PTY_TIMELINE=60 timeout -s KILL 300 python tools/tl_phases.py 18 2 2>&1 | tail -6
