"""Hottest CUDA source lines of an ncu report (source page, cuda+sass view):
python tools/ncu_src_hot.py REPORT.ncu-rep [N] -> stall-sample share and instructions executed per line."""
import csv, io, subprocess, sys
rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
data, fname = [], ""
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif len(r) > 8 and r[0].isdigit():
        try:
            data.append((int(r[4]), int(r[7]), f"{fname}:{r[0]}", r[1][:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
for s, e, loc, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% {e:>11d} {loc:<18s} {src}")
