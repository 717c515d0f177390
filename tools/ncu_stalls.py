"""Summarise an ncu --page source --csv (SASS) dump: top instructions by warp
stall samples and the stall-reason totals.  Usage: ncu_stalls.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
samp = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {s: 0.0 for s in stalls}
total = 0.0
for r in body:
    for s in stalls:
        try:
            tot[s] += float(r[ix[s]] or 0)
        except ValueError:
            pass
    try:
        total += float(r[samp] or 0)
    except ValueError:
        pass
print(f"kernel: {rows[0][1]}  total samples {total:.0f}")
for s, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {s:28s} {v:10.0f}  {100 * v / max(total, 1):5.1f}%")
body.sort(key=lambda r: -float(r[samp] or 0))
for r in body[:top]:
    print(f"  {float(r[samp] or 0):8.0f}  {r[ix['Address']]:>6s}  {r[ix['Source']][:90]}")
