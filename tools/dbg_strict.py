import sys; sys.path.insert(0,'.')
import numpy as np, oracle as O
from paper_2511_13905_b200 import api, synth
p = synth.SMALL["C1"](1)
d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t)
s=0.0
for i in range(p.n): s += gd[i]*p.grad[0][i]
print("expected ghat dot", repr(s), "alpha", info["alpha"], "wa*d0", info["alpha"]*d[0], flush=True)
with api.parity("strict"):
    st = api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values, p.bounds_g, p.is_eq, None, t=p.t)
print("ghat", st.g_hat, "Gmg", p.bounds_g - p.g_values, flush=True)
sx = p.x - p.x_prev; sy = p.g - p.g_prev
T = np.zeros((p.n, 6)); T[:,0]=sx*sx; T[:,1]=sx*sy; T[:,2]=sy*sy; T[:,3]=p.g*sy; T[:,4]=p.g_prev*p.g_prev
flat = T.reshape(-1)
acc=0.0
for e in range(p.n): acc += flat[2*e]
print("stale-layout hypothesis", acc)
gdv = info["alpha"]*d
acc=0.0
for e in range(p.n): acc += flat[2*e]
