"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
out, tot, fname = [], 0, ""
for r in rows:
    if r and r[0] == "File Path": fname = r[1]; continue
    if not r or not r[0] or r[0] == "Line No": continue
    try: s = int(r[iS]); n = int(r[iI])
    except (ValueError, IndexError): continue
    tot += s
    out.append((s, n, fname.split('/')[-1][:14] + ':' + r[0], r[1][:100]))
out.sort(reverse=True)
print("total samples", tot)
for s, n, ln, src in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/tot:5.1f}% {n:11d}  {ln:>20}  {src}")
