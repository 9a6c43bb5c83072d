"""Summarise an ncu --page source --csv dump: top source lines by stall samples."""
import csv, sys
rows = []
fname = None
hdr = None
for rec in csv.reader(open(sys.argv[1])):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] == "" or rec[0] == "Function Name":
        continue
    d = dict(zip(hdr, rec))
    try:
        samp = int(d["Warp Stall Sampling (All Samples)"])
    except (ValueError, KeyError):
        continue
    stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    top = sorted(stalls.items(), key=lambda x: -x[1])[:3]
    rows.append((samp, fname, rec[0], rec[1].strip()[:90], top))
tot = sum(r[0] for r in rows)
print("total samples", tot)
for samp, f, ln, src, top in sorted(rows, key=lambda r: -r[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*samp/tot:5.1f}% {f}:{ln} {src} | {top}")
