"""Dump controller-state snapshots (Plan bytes + the pass totals that follow)
from the host simulator for tools/ctlbench.cu (diagnostics)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import ctlsim
from paper_2511_13905_b200 import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
p = synth.CONFIGS[cfg](int(sys.argv[2]) if len(sys.argv) > 2 else 1)
rk = ctlsim.Rank(p, 0, p.n)
k = 0
while rk.phase() != ctlsim.PH_DONE:
    part = rk.partials()
    if rk.phase() in (1, 2):
        open(os.path.join(ROOT, f"tools/plan_{k}_ph{rk.phase()}.bin"), "wb").write(bytes(rk.plan))
        part.astype(np.float64).tofile(os.path.join(ROOT, f"tools/tot_{k}_ph{rk.phase()}.bin"))
    rk.consume(part)
    k += 1
print("passes", k, "plan bytes", len(bytes(rk.plan)))
