"""C5 on one GPU, stage by stage with timings (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_13905_b200 import api, synth, _lib

def log(*a):
    print(f"[{time.time() - T0:7.1f}s]", *a, flush=True)

T0 = time.time()
nz = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = synth.com_constrained(1024, 512, nz, 5)
log("generated n", p.n)
cu = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
X = [cu(getattr(p, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")]
A = cu(p.grad.reshape(-1))
out = {k: torch.empty(p.n, dtype=torch.float64, device="cuda") for k in ("x_new", "d", "rho_tilde")}
torch.cuda.synchronize()
log("on device")
structured = "--structured" in sys.argv
if structured:
    del A
    A = None
    prep = api.prepare_pgd_step(*X, None, p.g_values, p.bounds_g, p.is_eq, None, t=p.t, out=out,
                                rows=p.rows, grid=p.grid)
    log("structured rows")
step = (lambda: prep.run().result()) if structured else \
    (lambda: api.pgd_step(*X, A, p.g_values, p.bounds_g, p.is_eq, p.partition, t=p.t, out=out))
for it in range(3):
    t = time.time()
    r = step()
    torch.cuda.synchronize()
    log(f"step {it}: {1e3*(time.time()-t):.1f} ms path {r.projection.path.name} passes {r.projection.passes} "
        f"sweeps {r.projection.sweeps} newton {r.projection.newton_iters} y {r.y}")
if "--trace" in sys.argv:
    import ctypes as C
    ctx = _lib.context(0)
    ctx.lib.topt_b200_debug_trace(ctx.h, 1, None)
    step()
    buf = (C.c_ulonglong * 1024)()
    ctx.lib.topt_b200_debug_trace(ctx.h, 0, buf)
    allt = np.array(buf, dtype=np.float64).reshape(128, 8)
    tt = allt[:64]
    names = {0: "STEP", 1: "PREP", 2: "SWEEP", 3: "FEAS", 4: "NEWTON", 5: "FINAL", 7: "GATHER"}
    for k in range(64):
        if tt[k, 0] == 0:
            break
        print(f"pass {k:2d} {names.get(int(tt[k,5]),'?'):6s} start {1e-3*(tt[k,0]-tt[0,0]):9.1f} "
              f"body {1e-3*(tt[k,6]-tt[k,0]):8.1f} control {1e-3*(tt[k,4]-tt[k,3]):6.1f}")
log("done")
