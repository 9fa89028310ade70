"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv` output (stdin)."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = next(r for r in rows if r and r[0] == "Address")
i0 = rows.index(hdr)
data = [dict(zip(hdr, r)) for r in rows[i0 + 1:] if len(r) == len(hdr) and r[0] != "Address"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
agg = {s: sum(int(d[s] or 0) for d in data) for s in stalls}
print("by reason:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:8])
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[1]) if len(sys.argv) > 1 else 25]
for d in top:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    why = sorted(((int(d[k] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    print(f"{d['Address'][-5:]} {s:6d} {why} {d['Source'].strip()[:70]}")
