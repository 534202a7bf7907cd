"""Per-source-line stall samples / instructions / shared wavefronts from `ncu --page source --print-source cuda,sass --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 20 or r[0] in ("", "Line No"):
        continue
    try:
        ln = int(r[0])
        st, ins = float(r[4]), float(r[7])
        wf = float(r[19]) if r[19] not in ("-", "") else 0.0
    except ValueError:
        continue
    out.append((ins, st, wf, fname, ln, r[1].strip()[:80]))
ti = sum(o[0] for o in out)
ts = sum(o[1] for o in out)
print(f"total warp-instructions {ti:.3e}  stall samples {ts:.0f}")
for ins, st, wf, f, ln, src in sorted(out, key=lambda o: -o[1])[:n]:
    print(f"{f[:14]:14s}:{ln:4d} inst {100*ins/ti:5.1f}%  stall {100*st/ts:5.1f}%  smemW {wf/1e6:7.1f}M  {src}")
