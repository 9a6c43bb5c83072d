"""Top SASS instructions by stall samples from `ncu -i X --page source --csv --print-source=cuda,sass`."""
import csv, sys
seq = {}
cur = None
for rec in csv.reader(open(sys.argv[1])):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] not in ("", "Line No", "Function Name"):
        cur = f"{fname}:{rec[0]}"
        continue
    if rec[0] == "" and len(rec) > 4 and rec[2].startswith("0x"):
        try:
            n = int(rec[4])
        except ValueError:
            continue
        a = int(rec[2], 16)
        e = seq.setdefault(a, [n, rec[3].strip(), []])
        e[2].append(cur)
tot = sum(v[0] for v in seq.values())
print("total samples", tot)
for a, (n, s, srcs) in sorted(seq.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*n/tot:5.2f}% {hex(a)[-5:]} {s[:60]:60s} {srcs[-1]}")
