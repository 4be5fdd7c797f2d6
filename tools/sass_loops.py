"""List the loops (backward branches) of a cuobjdump -sass listing with their
instruction mix -- a quick look at what one iteration of a hot loop costs."""
import re, sys, collections
lines = open(sys.argv[1]).read().splitlines()
ins = []   # (addr, opcode, text)
for ln in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
    if not m:
        continue
    addr = int(m.group(1), 16)
    txt = m.group(2).strip()
    t = re.sub(r'^@!?U?P\w+\s+', '', txt)
    op = t.split()[0] if t else ''
    ins.append((addr, op, txt))
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k, (addr, op, txt) in enumerate(ins):
    if not op.startswith('BRA'):
        continue
    m = re.search(r'0x([0-9a-f]+)', txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= addr:
        continue
    body = [o for a, o, t in ins if tgt <= a <= addr]
    if len(body) < minlen:
        continue
    mix = collections.Counter(o.split('.')[0] for o in body)
    print(f"loop {tgt:#x}..{addr:#x}: {len(body)} instrs  " +
          " ".join(f"{o}:{c}" for o, c in mix.most_common(14)))
