"""Stall-reason totals and the hottest SASS lines of an ncu source-page CSV
(debug tool):  python scripts/ncu_source_stalls.py source.csv [top]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    for i in cols:
        tot[hdr[i]] += int(r[i] or 0)
    lines.append((int(r[2] or 0), r[1].strip(), {hdr[i]: int(r[i] or 0) for i in cols if int(r[i] or 0)}))
s = sum(tot.values())
print("samples", s)
for k, v in tot.most_common():
    if v:
        print(f"  {k:28s} {v / s:6.1%}")
op = collections.Counter()
for n, src, _ in lines:
    op[src.split()[0] if src else "?"] += n
print("by opcode:", ", ".join(f"{k} {v / s:.1%}" for k, v in op.most_common(12)))
for n, src, st in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{n / s:6.2%} {src[:60]:60s} {dict(sorted(st.items(), key=lambda x: -x[1])[:3])}")
