# debug: the C++ optimizer drop-in program hangs
set -x
O=gpurun_out/dbg_opt
mkdir -p $O
run() { name=$1; shift; env "$@" timeout 25 stdbuf -o0 -e0 ./tests/cpp/optimizer_ours > $O/$name.txt 2>&1; echo rc=$? >> $O/$name.txt; }
run default X=1
run multilaunch TOPT_B200_PERSISTENT=0 TOPT_B200_DEBUG_PHASES=1
run nostream TOPT_B200_STREAM=0
run blocking CUDA_LAUNCH_BLOCKING=1
timeout 60 python - > $O/py_dir.txt 2>&1 <<'P'
import ctypes as C, numpy as np, sys
sys.path.insert(0,'.')
from paper_2511_13905_b200 import _lib
ctx=_lib.context(0)
n=6000
rng=np.random.default_rng(0)
x=rng.random(n); xp=x+0.01*rng.standard_normal(n); g=-rng.random(n); gp=-rng.random(n)
d=np.empty(n); rt=np.empty(n)
a=C.c_double(); b=C.c_double(); fb=C.c_int32()
class S(C.Structure): _fields_=[(k,C.c_double) for k in ("alpha_max","alpha_fallback","omega","eps_alpha","tol_n")]+[("t_warmup",C.c_int32)]
s=S(1e2,0.2,1.0,1e-6,1e-6,50)
p=lambda v: v.ctypes.data_as(C.c_void_p)
print("calling", flush=True)
rc=ctx.lib.topt_b200_step_direction(ctx.h, n, p(x),p(xp),p(g),p(gp),p(gp),1,0.0,C.byref(s),p(d),p(rt),C.byref(a),C.byref(b),C.byref(fb))
print("rc",rc,a.value,b.value,fb.value, flush=True)
P
echo done
timeout 300 python -m pytest tests/test_gpu_upstream.py tests/test_gpu_fea.py -q --timeout 120 > $O/pytest_up.txt 2>&1
for c in C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
