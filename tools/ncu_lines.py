"""Warp-stall samples per CUDA source line from `ncu -i X --page source --csv --print-source cuda,sass`
(stdin): the SASS rows under each source row are summed.  Usage: ... | python tools/ncu_lines.py [top]"""
import csv
import sys
from collections import defaultdict

top = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 30
agg = defaultdict(lambda: [0, defaultdict(int), "", 0])
fname, cur, hdr = "", None, None
for r in csv.reader(sys.stdin):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:80])
        continue
    if cur is None or not r[2].startswith("0x"):
        continue
    d = dict(zip(hdr[2:], r[2:]))
    s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    a = agg[cur[:2]]
    a[0] += s
    a[2] = cur[2]
    ie = d.get("Instructions Executed", "0")
    a[3] += int(ie) if ie and ie not in ("-",) else 0
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v and v != "-":
            a[1][k[6:]] += int(v)
tot = sum(v[0] for v in agg.values())
print("total samples", tot, "instructions", sum(v[3] for v in agg.values()))
key = 3 if "--inst" in sys.argv else 0
for (f, ln), (s, st, src, ie) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    why = sorted(((v, k) for k, v in st.items()), reverse=True)[:2]
    print(f"{f}:{ln:5d} {s:6d} inst {ie:8d} {why} {src}")
