"""Count the SASS instructions of the coordinate-step loop of locus_warp_kernel<5,30,double>.

usage: python scripts/sass_loop.py [LIB] [--print]
The loop is located as the backward branch that encloses the ddot FMA tail (a run of DFMA
instructions accumulating into one register); prints its size and instruction mix.
"""
import collections, re, subprocess, sys

lib = next((a for a in sys.argv[1:] if not a.startswith("--")), "paper_2510_15649_b200/libladlasso_b200.so")
name = "_ZN3lad17locus_warp_kernelILi5ELi30EdEEvNS_9LocusArgsE"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
sec = out[out.index("Function : " + name):]
sec = sec[:sec.index("Function :", 20)] if "Function :" in sec[20:] else sec
ins = []
for line in sec.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = [a for a, _ in ins]
# the DFMA tail: the longest run of DFMA ... R2 instructions (allowing interleaved LDS)
best, run, start = (0, 0), 0, 0
for k, (a, t) in enumerate(ins):
    if t.startswith("DFMA"):
        if run == 0:
            start = k
        run += 1
        if run > best[1]:
            best = (start, run)
    elif not t.startswith("LDS"):
        run = 0
tail = best[0]
# enclosing loop: a backward BRA after the tail whose target precedes it, with the smallest span
loop = None
for k in range(tail, len(ins)):
    m = re.match(r"(@!?U?P\d+\s+)?BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", ins[k][1])
    if m and m.group(2):
        tgt = int(m.group(2), 16)
        if tgt < ins[tail][0]:
            loop = (addr.index(tgt) if tgt in addr else None, k)
            break
s, e = loop
body = ins[s:e + 1]
mix = collections.Counter(t.split()[0] if not t.startswith("@") else t.split()[1] for _, t in body)
print(f"loop {body[0][0]:#x}..{body[-1][0]:#x}: {len(body)} instructions (static, all paths)")
print(", ".join(f"{k} {v}" for k, v in mix.most_common(25)))
if "--print" in sys.argv:
    for a, t in body:
        print(f"{a:#07x} {t}")
