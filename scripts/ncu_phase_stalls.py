"""Stall samples of an ncu SASS source page attributed to kernel source lines
and phases (debug tool).  The SASS offsets are mapped to the outermost source
line with `nvdisasm -gi` of the library's cubin; phases are the kernel's
"// ==== <name>" banners.

    python scripts/ncu_phase_stalls.py source.csv lib.so k_stage_tmmaILi5E kernel.cuh [top]
"""
import collections, csv, os, re, subprocess, sys, tempfile

src_csv, lib, fn, cuh = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True, check=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
off2line, cur, on = {}, None, False
for ln in sass.splitlines():
    if ln.startswith(".text.") and fn in ln:
        on = True
        continue
    if on and ln.startswith(".text."):
        break
    if not on:
        continue
    if "//## File" in ln:
        cur = int(re.findall(r"line (\d+)", ln)[-1])
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        off2line[int(m.group(1), 16)] = cur
banners = [(i + 1, m.group(1)) for i, l in enumerate(open(cuh)) for m in [re.search(r"// =+ (.+?) =+", l)] if m]
def phase(line):
    name = "prologue"
    for b, n in banners:
        if line is not None and line >= b:
            name = n
    return name
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(rows[2][0], 16)
by_phase = collections.defaultdict(collections.Counter)
by_line = collections.defaultdict(collections.Counter)
total = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    line = off2line.get(int(r[0], 16) - base)
    for i in cols:
        v = int(r[i] or 0)
        by_phase[phase(line)][hdr[i]] += v
        by_line[line][hdr[i]] += v
        total += v
print("samples", total)
for p, c in by_phase.items():
    s = sum(c.values())
    print(f"{p:28s} {s / total:6.1%}  " + ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in c.most_common(5)))
src = open(cuh).read().splitlines()
for line, c in sorted(by_line.items(), key=lambda x: -sum(x[1].values()))[:top]:
    s = sum(c.values())
    txt = src[line - 1].strip()[:70] if line else "?"
    print(f"{s / total:6.2%} L{line} {txt:70s} " + ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in c.most_common(3)))
