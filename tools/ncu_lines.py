"""Aggregate ncu warp-stall samples by CUDA source line.

    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    cur_file = None
    hdr = None
    tot = {}
    total = 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 7:
            continue
        if r[0] != "":  # a source line row (aggregated over its SASS)
            try:
                s = int(r[4])
            except ValueError:
                continue
            key = (cur_file, int(r[0]), r[1][:70])
            tot[key] = tot.get(key, 0) + s
            total += s
    print("total samples", total)
    for (f, ln, src), s in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{100.0 * s / max(total, 1):5.1f}% {s:7d} {f}:{ln} {src}")


if __name__ == "__main__":
    main()
