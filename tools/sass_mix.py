"""Static SASS opcode mix of one kernel in a cubin: python tools/sass_mix.py X.cubin <kernel-substring>."""
import collections, re, subprocess, sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
cur, mix = None, collections.Counter()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur and sys.argv[2] in cur:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            mix[m.group(2)] += 1
tot = sum(mix.values())
print("total", tot)
for k, v in mix.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{k:12s} {v:6d}")
