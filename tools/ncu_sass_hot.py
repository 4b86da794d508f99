"""Hottest SASS instructions of an ncu report's source page (--print-source sass):
python tools/ncu_sass_hot.py REPORT.ncu-rep [N] -> stall samples / instructions executed per SASS line,
plus totals by opcode."""
import collections, csv, io, subprocess, sys
rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iS] or 0), int(r[iE] or 0), r[iSrc].strip(), r[0]))
    except (ValueError, IndexError):
        pass
tot_s = sum(d[0] for d in data) or 1
tot_e = sum(d[1] for d in data) or 1
print(f"total stall samples {tot_s}, instructions executed {tot_e}")
by = collections.Counter()
byc = collections.Counter()
for s, e, src, _ in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    by[op] += s
    byc[op] += e
print("by opcode (samples%, instr%):")
for op, s in by.most_common(25):
    print(f"  {op:12s} {100*s/tot_s:5.1f}% {100*byc[op]/tot_e:5.1f}%")
print("hottest lines:")
for s, e, src, addr in sorted(data, reverse=True)[:n]:
    print(f"  {100*s/tot_s:5.2f}% {e:>10d} {addr[-5:]} {src[:90]}")
