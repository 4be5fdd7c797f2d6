"""Where does the host-buffer step time go?  (diagnostics)"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2511_13905_b200 import api, synth

p = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"](2)
n = p.n
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
H = [pin(getattr(p, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")] + [pin(p.grad.reshape(-1))]
D = [torch.empty_like(h, device="cuda") for h in H]
HO = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
torch.cuda.synchronize()
s = torch.cuda.current_stream()
for rep in range(3):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for h, d in zip(H, D):
        d.copy_(h, non_blocking=True)
    e1.record()
    HO[0].copy_(D[0], non_blocking=True); HO[1].copy_(D[1], non_blocking=True)
    e2.record(); torch.cuda.synchronize()
    nb = sum(h.numel() * 8 for h in H)
    print(f"H2D {nb/1e6:.1f} MB {e0.elapsed_time(e1):.3f} ms ({nb/e0.elapsed_time(e1)/1e6:.1f} GB/s)  "
          f"D2H 16.8 MB {e1.elapsed_time(e2):.3f} ms ({16.777e6/e1.elapsed_time(e2)/1e6:.1f} GB/s)")
# concurrent H2D + D2H
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); e0.record()
with torch.cuda.stream(s2):
    HO[0].copy_(D[0], non_blocking=True); HO[1].copy_(D[1], non_blocking=True)
for h, d in zip(H, D):
    d.copy_(h, non_blocking=True)
s.wait_stream(s2); e1.record(); torch.cuda.synchronize()
print(f"H2D+D2H concurrent: {e0.elapsed_time(e1):.3f} ms")
hx = [h.numpy() for h in H]
out = {"x_new": HO[0].numpy(), "d": HO[1].numpy()}
for rep in range(5):
    t0 = time.perf_counter()
    api.pgd_step(*hx[:5], hx[5], p.g_values, p.bounds_g, p.is_eq, p.partition, t=p.t,
                 host_outputs=("x_new", "d"), out=out)
    t1 = time.perf_counter()
    print(f"api.pgd_step host call: {1e3*(t1-t0):.3f} ms")
from paper_2511_13905_b200 import _lib
ctx = _lib.context(0)
ctx.set_profiling(True)
ctx.kernel_time()
for rep in range(3):
    t0 = time.perf_counter()
    api.pgd_step(*hx[:5], hx[5], p.g_values, p.bounds_g, p.is_eq, p.partition, t=p.t,
                 host_outputs=("x_new", "d"), out=out)
    t1 = time.perf_counter()
    print(f"host call {1e3*(t1-t0):.3f} ms; kernel (launch->end on the stream) {ctx.kernel_time()}")
ctx.set_profiling(False)
