"""Full-size GPU parity spot check for one config (diagnostics; the pytest
suite runs the same checks): oracle vs the B200 path on the same inputs."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from paper_2511_13905_b200 import api, synth
from test_gpu_parity import check_projection

for name in sys.argv[1:]:
    p = synth.CONFIGS[name]()
    t0 = time.time()
    res, orc = check_projection(p)
    print(name, "path", orc["path"], "iters", orc.get("newton_iters"), orc.get("bisect_iters"),
          "gpu passes", res.passes, "sweeps", res.sweeps, "near_ties", res.near_ties,
          f"ok ({time.time() - t0:.1f} s)", flush=True)
