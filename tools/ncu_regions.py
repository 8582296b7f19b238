#!/usr/bin/env python3
"""Group an ncu source-page (SASS) capture into straight-line regions by execution count and
print where the warp-stall samples go.  usage: ncu_regions.py REPORT [launch-index] [min-samples]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; skip = sys.argv[2] if len(sys.argv) > 2 else "0"; mins = float(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][1] if len(rows[0]) > 1 else rows[0])
h = rows[1]; data = rows[2:]
g = lambda r, k: r[h.index(k)]
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
seen = set(); lst = []
for r in data:
    a = g(r, "Address")
    if a in seen: continue
    seen.add(a)
    try:
        ex = float(g(r, "Instructions Executed") or 0); s = float(g(r, "Warp Stall Sampling (All Samples)") or 0)
    except (ValueError, IndexError):
        continue
    lst.append((int(a, 16), g(r, "Source").strip(), ex, s, {c: float(g(r, c) or 0) for c in cols}))
lst.sort()
tot = sum(x[3] for x in lst); texec = sum(x[2] for x in lst)
print("total samples", tot, "instructions", len(lst), "warp-instr executed %.3gM" % (texec / 1e6))
cur = None; out = []
for a, src, ex, s, st in lst:
    if int(ex) != cur:
        if cur is not None: out.append(blk)
        cur = int(ex); blk = [a, 0, cur, 0.0, {}, src]
    blk[1] += 1; blk[3] += s
    for c, v in st.items(): blk[4][c] = blk[4].get(c, 0) + v
out.append(blk)
for a, n, ex, acc, stl, src in out:
    if acc >= mins:
        top = sorted(stl.items(), key=lambda kv: -kv[1])[:3]
        print("%6x n=%3d exec=%7d samples=%4d %4.1f%%" % (a & 0xfffff, n, ex, acc, 100 * acc / tot),
              [(k[6:], int(v)) for k, v in top], src[:40])
