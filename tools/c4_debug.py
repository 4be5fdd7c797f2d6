import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2511_13905_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = synth.CONFIGS[name](seed)
ref = O.pgd_step(p)
rt, gd = ref["rho_tilde"], ref["gd_step"]
lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition)
print("ghat gpu", lin.g_hat)
print("ghat ref", ref["ghat"])
res = api.project(rt, lin, p.lower, p.upper)
orc = O.project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition, p.lower, p.upper)
print("path", res.path.name, orc["path"], "iters", res.newton_iters, orc["newton_iters"], "stage1", getattr(res, "stage1_row", None), orc.get("stage1_row"))
print("y gpu", res.y)
print("y ref", orc["y"])
print("conv", res.converged, orc["converged"], "resid", res.residual, orc["residual"])
for k in ("gammas", "phi_inf", "trace"):
    if k in orc: print(k, orc[k])
print("res fields", [a for a in dir(res) if not a.startswith("_")])
x_g = rt + res.delta
x_o = rt + orc["delta"]
print("x normwise rel", np.max(np.abs(x_g - x_o)) / np.max(np.abs(x_o)))
print("y abs diff", np.abs(res.y - orc["y"]))
def masks(y):
    z = np.zeros(p.n)
    for j in range(p.m):
        if y[j] != 0.0: z = z + y[j] * p.grad[j]
    return np.where(z < p.lower - rt, 1, np.where(z > p.upper - rt, 2, 0))
print("mask diffs", int(np.count_nonzero(masks(res.y) != masks(orc["y"]))))
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/{name}_{seed}_gpu.npz", y=res.y, delta=res.delta, iters=res.newton_iters)
