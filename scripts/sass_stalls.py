"""Summarise an `ncu --page source --csv --print-source sass` dump: stall samples by reason and by
instruction opcode, and the top stalled instructions (the first kernel of a multi-kernel dump).
usage: sass_stalls.py dump.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = {r: h.index(r) for r in reasons}
si, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
by_reason = collections.Counter()
by_op = collections.Counter()
by_op_reason = collections.defaultdict(collections.Counter)
insts = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":  # a multi-kernel dump: the first kernel only
        break
    if len(r) < len(h):
        continue
    src = r[si].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    tot = float(r[ai] or 0)
    by_op[op] += tot
    for k, i in ri.items():
        v = float(r[i] or 0)
        by_reason[k] += v
        by_op_reason[op][k] += v
    insts.append((tot, src, {k: float(r[i] or 0) for k, i in ri.items() if float(r[i] or 0) > 0}))
T = sum(by_reason.values())
print("samples", T)
for k, v in by_reason.most_common():
    if v:
        print(f"  {k:24s} {v:8.0f} {100 * v / T:5.1f}%")
print("by opcode:")
for k, v in by_op.most_common(12):
    print(f"  {k:10s} {v:8.0f} {100 * v / T:5.1f}%  ", dict(by_op_reason[k].most_common(4)))
print("top instructions:")
for tot, src, d in sorted(insts, key=lambda x: -x[0])[:top]:
    print(f"  {tot:6.0f}  {src[:60]:60s} {dict(sorted(d.items(), key=lambda x: -x[1])[:3])}")
