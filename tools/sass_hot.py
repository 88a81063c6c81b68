"""Print the hot SASS lines of one kernel from `ncu --page source --csv --print-source sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
for b in blocks[:1]:
    h = b["hdr"]
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = b["rows"]
    tot = sum(int(r[iE] or 0) for r in data)
    totw = sum(int(r[iW] or 0) for r in data)
    print(b["name"][:100], "inst", tot, "samples", totw)
    for r in data:
        e, w = int(r[iE] or 0), int(r[iW] or 0)
        if e > tot * frac or w > totw * 2 * frac:
            print(f"{r[0][-5:]} {e:>11d} {w:>6d}  {r[iS].strip()[:90]}")

if len(sys.argv) > 3:  # top-N by stall samples
    b = blocks[0]
    h = b["hdr"]
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    rows = sorted(b["rows"], key=lambda r: -int(r[iW] or 0))[: int(sys.argv[3])]
    print("--- top by samples")
    for r in sorted(rows, key=lambda r: r[0]):
        print(f"{r[0][-5:]} {int(r[iE] or 0):>11d} {int(r[iW] or 0):>6d}  {r[iS].strip()[:90]}")
