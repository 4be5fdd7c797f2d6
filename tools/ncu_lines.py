"""Attribute an ncu SASS-level stall profile of k_step to source lines
(diagnostics).  ncu's source page lists k_step's instructions in order; the
cubin disassembly with line info (nvdisasm --print-line-info) gives the
source line of instruction k.  Usage:
  python tools/ncu_lines.py <report.ncu-rep> <lines.sass> [function-substring]"""
import csv, re, subprocess, sys, collections

rep, lines_path = sys.argv[1], sys.argv[2]
fn = sys.argv[3] if len(sys.argv) > 3 else "k_step"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) > 3]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iX = hdr.index("Instructions Executed")
# instruction k -> (file, line)
src = []
cur = ("?", 0); inside = False
for ln in open(lines_path):
    if ln.startswith("//----") and ".text." in ln:
        inside = fn in ln
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln):
        src.append(cur)
print("sass rows", len(data), "disasm instrs", len(src))
agg = collections.Counter(); exe = collections.Counter()
for k, r in enumerate(data):
    key = src[k] if k < len(src) else ("?", 0)
    agg[key] += float(r[iS] or 0); exe[key] += float(r[iX] or 0)
tot = sum(agg.values())
print(f"total samples {tot:.0f}")
for key, v in agg.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    print(f"{100*v/tot:5.1f}%  {key[0]}:{key[1]}  exec {exe[key]:.0f}")
