"""World-size-2 test of the sharded path on CPU (gloo): each rank owns a
contiguous element slab, computes its pass partials, the partials are
all-gathered and combined in fixed rank order, and every rank runs the
controller redundantly; decisions must be identical on both ranks and the
result must equal the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PMAX = 512


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, seed, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import ctlsim
    import oracle as O
    from paper_2511_13905_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.SMALL[name](seed)
    ref = O.pgd_step(p)
    lo, hi = ctlsim.bounds(p.n, world)[rank]
    rk = ctlsim.Rank(p, lo, hi, ctlsim.JOB_PROJECT, ref["rho_tilde"], ref["gd_step"], ref["ghat"])
    passes = 0
    while rk.phase() != ctlsim.PH_DONE:
        part = rk.partials()
        ns = part.size
        buf = torch.zeros(PMAX, dtype=torch.float64)
        buf[:ns] = torch.from_numpy(part)
        gathered = [torch.zeros(PMAX, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, buf)
        tot = ctlsim.combine([g[:ns].numpy() for g in gathered], rk.ops(ns))
        rk.consume(tot)
        passes += 1
    res = rk.result(p.m)
    ys = [torch.zeros(p.m, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(ys, torch.from_numpy(res["y"]))
    if rank == 0:
        orc = O.project(ref["rho_tilde"], p.grad, p.g_values, p.bounds_g, ref["gd_step"],
                        p.is_eq, p.partition)
        q.put(dict(y=res["y"], y_ranks=[t.numpy() for t in ys], path=res["path"],
                   orc_y=orc["y"], orc_path=orc["path"], passes=passes))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C2", "C3", "C4p"])
def test_two_rank_gloo(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, 3, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.array_equal(out["y_ranks"][0], out["y_ranks"][1])
    assert out["path"] == out["orc_path"]
    if out["path"] == "newton":
        np.testing.assert_allclose(out["y"], out["orc_y"], rtol=1e-9, atol=1e-9)
    else:
        assert np.array_equal(out["y"], out["orc_y"])
