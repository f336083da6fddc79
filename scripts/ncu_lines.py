"""Per-source-line dynamic instruction counts of one kernel from an ncu capture.

usage: python scripts/ncu_lines.py REP.ncu-rep LIB.so KERNEL_MANGLED [--top N] [--per X]
Joins ncu's SASS source page ("Instructions Executed" per address) with the line
table of `nvdisasm -g` on the library's cubin (offsets within the kernel's text
section), and prints instructions executed per (file, line), optionally divided by X
(e.g. the number of coordinate steps of the launch)."""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, lib, kern = sys.argv[1:4]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 60
per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
cols = rows[hdr]
ia, ie = cols.index("Address"), cols.index("Instructions Executed")
samp = cols.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ia], 16), float(r[ie] or 0), float(r[samp] or 0)) for r in rows[hdr + 1:] if r and r[0].startswith("0x")]
base = data[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
sec = sass[sass.index(".text." + kern + ":"):]
nxt = sec.find("//---------------------", 10)
sec = sec[:nxt] if nxt > 0 else sec
where = {}
chain_of = {}
text_of = {}
cur = ("?", 0)
chain = []
pending = []
for line in sec.splitlines():
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', line)
    if m:
        fr = [(os.path.basename(m.group(1)), int(m.group(2)))]
        fr += [(os.path.basename(a), int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        pending.append(fr)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", line)
    if m:
        text_of[int(m.group(1), 16)] = m.group(2).strip()
        if pending:
            chain = max(pending, key=len)  # the innermost entry carries the full inline chain
            cur = chain[0]
            pending = []
        where[int(m.group(1), 16)] = cur
        chain_of[int(m.group(1), 16)] = chain
acc = collections.Counter()
stall = collections.Counter()
tot = 0.0
for a, n, s in data:
    k = where.get(a - base, ("?", 0))
    acc[k] += n
    stall[k] += s
    tot += n
print(f"total instructions executed {tot:.4g} ({tot / per:.1f} per unit)")
if "--buckets" in sys.argv:
    # bucket = the first rule whose (file, first, last) range contains any frame of the inline chain
    rules = [tuple(x.split(":")) for x in sys.argv[sys.argv.index("--buckets") + 1].split(",")]
    bk = collections.Counter()
    shown = collections.Counter()
    for a, n, _ in data:
        ch = chain_of.get(a - base, [])
        name = "other"
        for nm, f, lo, hi in rules:
            if any(fr[0] == f and int(lo) <= fr[1] <= int(hi) for fr in ch):
                name = nm
                break
        bk[name] += n
        if "--show" in sys.argv and name == sys.argv[sys.argv.index("--show") + 1]:
            shown[tuple(ch)] += n
    for nm, n in bk.most_common():
        print(f"  bucket {nm:14s} {n / per:8.2f} per unit  {100 * n / tot:5.1f}%")
    for ch, n in shown.most_common(25):
        print(f"    {n / per:7.2f}  " + " <- ".join(f"{f}:{l}" for f, l in ch))
if "--sass-top" in sys.argv:  # the hottest SASS instructions: offset, count per unit, source line, text
    nsass = int(sys.argv[sys.argv.index("--sass-top") + 1])
    for a, n, smp in sorted(data, key=lambda x: -x[1])[:nsass]:
        off = a - base
        f, l = where.get(off, ("?", 0))
        print(f"  sass {off:#08x} {n / per:7.3f} samples {smp:7.0f}  {f}:{l}  {text_of.get(off, '?')}")
for (f, l), n in acc.most_common(top):
    print(f"{n / per:8.2f} {100 * n / tot:5.1f}%  stall-samples {stall[(f, l)]:8.0f}  {f}:{l}")
