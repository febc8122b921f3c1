"""Stall-reason totals per source file:line range from an ncu source CSV."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
want = sys.argv[2:]  # e.g. trg_assoc.cuh:20-90
tot = collections.Counter(); fname = ""
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split('/')[-1]; continue
    if not r or not r[0] or r[0] == "Line No" or len(r) < len(hdr): continue
    try: ln = int(r[0])
    except ValueError: continue
    ok = not want
    for w in want:
        f, rg = w.split(':'); a, b = map(int, rg.split('-'))
        if fname == f and a <= ln <= b: ok = True
    if not ok: continue
    for i in cols:
        try: tot[hdr[i]] += int(r[i])
        except ValueError: pass
s = sum(tot.values())
for k, v in tot.most_common(12): print(f"{k:28s} {v:8d} {100*v/max(s,1):5.1f}%")
