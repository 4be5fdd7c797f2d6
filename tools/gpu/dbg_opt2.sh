set -x
O=gpurun_out/dbg_opt2
mkdir -p $O
cat > /tmp/pydir.py <<'P'
import ctypes as C, numpy as np, sys, os
sys.path.insert(0,'.')
from paper_2511_13905_b200 import _lib
ctx=_lib.context(0)
n=int(sys.argv[1])
rng=np.random.default_rng(0)
x=rng.random(n); xp=x+0.01*rng.standard_normal(n); g=-rng.random(n); gp=-rng.random(n)
d=np.empty(n); rt=np.empty(n)
a=C.c_double(); b=C.c_double(); fb=C.c_int32()
class S(C.Structure): _fields_=[(k,C.c_double) for k in ("alpha_max","alpha_fallback","omega","eps_alpha","tol_n")]+[("t_warmup",C.c_int32)]
s=S(1e2,0.2,1.0,1e-6,1e-6,50)
p=lambda v: v.ctypes.data_as(C.c_void_p)
print("calling", n, flush=True)
rc=ctx.lib.topt_b200_step_direction(ctx.h, n, p(x),p(xp),p(g),p(gp),p(gp),1,0.0,C.byref(s),p(d),p(rt),C.byref(a),C.byref(b),C.byref(fb))
print("rc",rc,a.value,b.value,fb.value, flush=True)
P
for n in 6000 6144 1048576 100000; do timeout 30 python /tmp/pydir.py $n > $O/py_$n.txt 2>&1; echo rc=$? >> $O/py_$n.txt; done
TOPT_B200_COMPACT=0 timeout 30 python /tmp/pydir.py 6000 > $O/py_nocompact.txt 2>&1; echo rc=$? >> $O/py_nocompact.txt
timeout 120 compute-sanitizer --tool memcheck python /tmp/pydir.py 6000 > $O/memcheck.txt 2>&1; echo rc=$? >> $O/memcheck.txt
echo done
