"""Executed FP32 flops of one kernel from an ncu source page (SASS level):
python tools/sass_flops.py <page.csv> <gpu_time_s> <positions_per_launch>

Counts every FP32 arithmetic SASS instruction by its thread-instruction count
(predicated-on): FFMA 2 flops, FADD/FMUL 1, FFMA2 4, FADD2/FMUL2 2 (the packed
sm_100 forms do two lanes per thread), MUFU 1."""
import csv, json, re, sys

FLOPS = {"FFMA": 2, "FADD": 1, "FMUL": 1, "FFMA2": 4, "FADD2": 2, "FMUL2": 2, "MUFU": 1,
         "FMNMX": 0, "FSETP": 0}
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
ia = hdr.index("Source")
ic = hdr.index("Predicated-On Thread Instructions Executed")
tot = {}
for r in rows:
    if len(r) <= ic or not r[0].startswith("0x"):
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ia])
    if not m:
        continue
    op = m.group(2)
    try:
        n = int(r[ic].replace(",", ""))
    except ValueError:
        continue
    tot[op] = tot.get(op, 0) + n
flops = sum(FLOPS.get(k, 0) * v for k, v in tot.items())
t = float(sys.argv[2])
pos = int(sys.argv[3])
out = {"executed_fp32_flop_per_launch": flops, "executed_fp32_tflops": flops / t / 1e12,
       "per_position_mflop": flops / pos / 1e6,
       "thread_instructions": {k: tot[k] for k in sorted(tot, key=lambda k: -tot[k])[:16]}}
print(json.dumps(out, indent=1))
