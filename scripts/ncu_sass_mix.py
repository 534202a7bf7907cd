"""Per-kernel SASS instruction mix and hottest stall sites from an ncu report (source page)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # e.g. rows per launch
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kern, data, hdr = None, [], None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        kern = r[1]
        data.append((kern, []))
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and kern:
        data[-1][1].append(dict(zip(hdr, r)))
for k, v in data:
    tot = sum(int(x["Instructions Executed"] or 0) for x in v)
    samp = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in v)
    print(f"== {k[:100]}\n   warp-instructions {tot:,}  per unit {tot / units:.1f}  stall samples {samp}")
    c = Counter()
    for x in v:
        op = x["Source"].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(x["Instructions Executed"] or 0)
    print("   mix:", ", ".join(f"{o} {n / units:.1f}" for o, n in c.most_common(18)))
    hot = sorted(v, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:8]
    for x in hot:
        print(f"   hot {int(x['Warp Stall Sampling (All Samples)']):7d}  {x['Source'].strip()[:90]}")
