"""Instruction mix (warp instructions executed per opcode) of the first kernel
in an `ncu --page source --csv --print-source sass` dump."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address" and hdr is None:
        hdr = r
    elif hdr is not None and len(r) == len(hdr):
        if r[0] == "Address":
            break
        data.append(r)
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
mix = collections.Counter()
for r in data:
    op = r[iS].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    mix[o.split(".")[0]] += int(r[iE] or 0)
tot = sum(mix.values())
print(f"total {tot / 1e6:.1f} M")
for o, c in mix.most_common(40):
    print(f"{o:10s} {c / 1e6:8.1f} M  {100 * c / tot:5.1f} %")
