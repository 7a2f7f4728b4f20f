"""Attribute ncu SASS-level samples / executed instructions to CUDA source lines.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [top] [opcode-regex]
(with an opcode regex, e.g. "IMAD|FSEL", also prints that opcode class's share per line)
Needs the .so compiled with -lineinfo (it is) and nvdisasm/cuobjdump in PATH.
"""
import csv, io, re, subprocess, sys, collections, tempfile, os

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
opre = re.compile(sys.argv[4]) if len(sys.argv) > 4 else None
so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2401_13680_b200", "libpastila.so")
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "-c", "1", "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1]
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
sass = []
for r in rows[2:]:
    try:
        sass.append((int(r[ia], 16), int(r[iw] or 0), int(r[ie] or 0), r[isrc]))
    except Exception:
        pass
# line info from nvdisasm of the matching function
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
addr2line = {}
mang = None
for cb in cubins:
    txt = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    cur = None; line = None
    for ln in txt.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur and re.search(kre, cur):
            addr2line[(cur, int(m.group(1), 16))] = line
funcs = sorted({f for f, _ in addr2line})
# match the template arguments of the profiled kernel, e.g. "<(int)5, (int)256, (int)5>"
# mangled name of the profiled instantiation, e.g. "8k_mpdistILi5ELi256ELi5EiE"
mb = re.search(r"::(\w+)<(.*)>\(", kname) or re.search(r"(\w+)<(.*)>\(", kname)
want = None
if mb:
    enc = []
    for t in [a.strip() for a in mb.group(2).split(",")]:
        mi = re.match(r"\(int\)(-?\d+)", t)
        mb2 = re.match(r"\(bool\)(\d)", t)
        enc.append(f"Li{mi.group(1)}E" if mi else f"Lb{mb2.group(1)}E" if mb2 else {"int": "i", "double": "d"}.get(t, ""))
    want = f"{len(mb.group(1))}{mb.group(1)}I{''.join(enc)}E"
cands = [f for f in funcs if want and want in f] or funcs
best = None
for f in cands:
    n = sum(1 for (ff, _) in addr2line if ff == f)
    if best is None or abs(n - len(sass)) < abs(best[1] - len(sass)):
        best = (f, n)
f = best[0]
agg = collections.defaultdict(lambda: [0, 0, 0])
tot_w = sum(s[1] for s in sass) or 1
tot_e = sum(s[2] for s in sass) or 1
base = sass[0][0]
for i, (a, w, e, src) in enumerate(sass):
    key = addr2line.get((f, a - base), ("?", -1))
    agg[key][0] += w
    agg[key][1] += e
    if opre is not None:
        t = src.strip().split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else ""))
        if opre.search(op):
            agg[key][2] += e
print(f"kernel {kname}  ({len(sass)} SASS instrs; function {f})")
srcfile = {}
for (fn, ln), (w, e, oe) in sorted(agg.items(), key=lambda t: -(t[1][2] if opre is not None else t[1][0]))[:top]:
    if fn not in srcfile:
        p = os.path.join(os.path.dirname(so), "csrc", fn)
        srcfile[fn] = open(p).read().splitlines() if os.path.exists(p) else []
    text = srcfile[fn][ln - 1].strip() if 0 < ln <= len(srcfile[fn]) else ""
    extra = f" {100*oe/tot_e:5.1f}% op" if opre is not None else ""
    print(f"{100*w/tot_w:5.1f}% stall {100*e/tot_e:5.1f}% inst{extra}  {fn}:{ln:<4d} {text[:90]}")
