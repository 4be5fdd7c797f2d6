"""ctypes binding of libtopt_b200.so (include/topt_b200.h).

The shared library is built in-tree by ``paper_2511_13905_b200.build.build()``
(``nvcc -gencode arch=compute_100a,code=sm_100a``).  There is no fallback:
if the library or a CUDA device is missing every call raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtopt_b200.so")

MAX_M = 16

OK = 0
ERR_PARAMETER, ERR_DOMAIN, ERR_SINGULAR, ERR_INFEASIBLE, ERR_NUMERICAL, ERR_UNSUPPORTED, \
    ERR_CUDA, ERR_INTERNAL = range(1, 9)

PROJECT_AUTO, PROJECT_SINGLE, PROJECT_INDEPENDENT, PROJECT_NEWTON = range(4)

_dp = C.POINTER(C.c_double)


class ProjOptions(C.Structure):
    _fields_ = [("c", C.c_double), ("tol_b", C.c_double), ("tol_n", C.c_double),
                ("newton_maxiter", C.c_int32), ("binary_maxiter", C.c_int32)]


class PgdSettingsC(C.Structure):
    _fields_ = [("alpha_max", C.c_double), ("alpha_fallback", C.c_double),
                ("omega", C.c_double), ("eps_alpha", C.c_double), ("tol_n", C.c_double),
                ("t_warmup", C.c_int32)]


class ProjMeta(C.Structure):
    _fields_ = [("path", C.c_int32), ("newton_iters", C.c_int32), ("converged", C.c_int32),
                ("curvature_violations", C.c_int32), ("residual", C.c_double),
                ("passes", C.c_int32), ("sweeps", C.c_int32), ("stage1_row", C.c_int32),
                ("near_ties", C.c_int32), ("min_margin", C.c_double),
                ("bisect_iters", C.c_int32 * MAX_M), ("alpha", C.c_double),
                ("beta", C.c_double), ("fallback", C.c_int32), ("local_sweeps", C.c_int32),
                ("gathered", C.c_int32), ("exact_passes", C.c_int32), ("active", C.c_double)]


class Linearization(C.Structure):
    _fields_ = [("num_constraints", C.c_size_t), ("num_vars", C.c_size_t),
                ("grad", C.c_void_p), ("g_values", C.c_void_p), ("bounds_g", C.c_void_p),
                ("gd_step", C.c_void_p), ("g_hat", C.c_void_p), ("g_hat_err", C.c_void_p),
                ("is_equality", C.c_void_p), ("part_offsets", C.c_void_p),
                ("part_indices", C.c_void_p), ("owner", C.c_void_p)]


class StepProblem(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int32), ("t", C.c_int32),
                ("violation", C.c_double), ("lower", C.c_double), ("upper", C.c_double),
                ("x", C.c_void_p), ("x_prev", C.c_void_p), ("g", C.c_void_p),
                ("g_prev", C.c_void_p), ("d_prev", C.c_void_p), ("grad", C.c_void_p),
                ("g_values", C.c_void_p), ("bounds_g", C.c_void_p),
                ("is_equality", C.c_void_p), ("part_offsets", C.c_void_p),
                ("part_indices", C.c_void_p), ("owner", C.c_void_p)]


class StepOutputs(C.Structure):
    _fields_ = [("x_new", C.c_void_p), ("d", C.c_void_p), ("rho_tilde", C.c_void_p),
                ("delta", C.c_void_p), ("y", C.c_void_p), ("slacks", C.c_void_p),
                ("g_hat", C.c_void_p), ("mask", C.c_void_p)]


EXPORTS = [
    "topt_b200_version", "topt_b200_ctx_create", "topt_b200_ctx_destroy",
    "topt_b200_last_error", "topt_b200_kernel_launches", "topt_b200_get_stream",
    "topt_b200_set_stream", "topt_b200_default_options", "topt_b200_default_settings",
    "topt_b200_build", "topt_b200_delta_of_y", "topt_b200_constraint_residual_h",
    "topt_b200_project", "topt_b200_project_dev", "topt_b200_owner_map",
    "topt_b200_pgd_step", "topt_b200_pgd_step_dev", "topt_b200_step_direction",
    "topt_b200_set_profiling", "topt_b200_kernel_time", "topt_b200_step_time",
    "topt_b200_debug_trace",
    "topt_b200_nccl_unique_id", "topt_b200_ctx_create_ranks", "topt_b200_pgd_step_ranks",
    "topt_b200_set_structured_rows", "topt_b200_set_parity", "topt_b200_get_parity",
    "topt_b200_filter_create", "topt_b200_filter_destroy", "topt_b200_filter_nnz",
    "topt_b200_filter_csr", "topt_b200_filter_apply", "topt_b200_filter_apply_dev",
    "topt_b200_csr_apply", "topt_b200_interpolate_stiffness_dev",
    "topt_b200_element_stiffness_q4", "topt_b200_compliance_gradient_dev",
    "topt_b200_ctx_create_lockstep", "topt_b200_pgd_step_lockstep", "topt_b200_fe_solve_dev",
]

_lib = None


def load():
    """Load libtopt_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with paper_2511_13905_b200.build.build() "
            "(no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    lib.topt_b200_version.restype = C.c_char_p
    lib.topt_b200_last_error.restype = C.c_char_p
    lib.topt_b200_last_error.argtypes = [C.c_void_p]
    lib.topt_b200_kernel_launches.restype = C.c_int64
    lib.topt_b200_kernel_launches.argtypes = [C.c_void_p]
    lib.topt_b200_get_stream.restype = C.c_void_p
    lib.topt_b200_get_stream.argtypes = [C.c_void_p]
    lib.topt_b200_ctx_destroy.argtypes = [C.c_void_p]
    lib.topt_b200_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    vp, d, i32, i64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
    sig = {
        "topt_b200_build": [vp, vp, vp, vp],
        "topt_b200_delta_of_y": [vp, vp, vp, vp, d, d, vp],
        "topt_b200_constraint_residual_h": [vp, vp, vp, vp, d, d, d, vp],
        "topt_b200_project": [vp, C.c_int, vp, vp, d, d, vp, vp, vp, vp, vp],
        "topt_b200_project_dev": [vp, C.c_int, vp, vp, d, d, vp, vp, vp, vp, vp, vp],
        "topt_b200_owner_map": [vp, i64, i32, vp, vp, vp],
        "topt_b200_pgd_step": [vp, vp, vp, vp, vp, vp],
        "topt_b200_pgd_step_dev": [vp, vp, vp, vp, vp, vp],
        "topt_b200_set_stream": [vp, vp],
        "topt_b200_step_direction": [vp, i64, vp, vp, vp, vp, vp, i32, d, vp, vp, vp, vp, vp,
                                     vp],
        "topt_b200_set_profiling": [vp, C.c_int],
        "topt_b200_debug_trace": [vp, C.c_int, vp],
        "topt_b200_kernel_time": [vp, vp, vp, vp],
        "topt_b200_step_time": [vp, vp, vp, vp],
        "topt_b200_nccl_unique_id": [vp, C.c_size_t],
        "topt_b200_ctx_create_ranks": [C.c_int, C.c_int, C.c_int, vp, C.POINTER(C.c_void_p)],
        "topt_b200_pgd_step_ranks": [vp, vp, i64, vp, vp, vp, vp, vp],
        "topt_b200_default_options": [vp],
        "topt_b200_set_structured_rows": [vp, i32, vp, vp, i64],
        "topt_b200_default_settings": [vp],
        "topt_b200_set_parity": [vp, C.c_int],
        "topt_b200_get_parity": [vp],
        "topt_b200_filter_create": [vp, i32, i32, d, C.POINTER(C.c_void_p)],
        "topt_b200_filter_csr": [vp, vp, vp, vp],
        "topt_b200_filter_apply": [vp, vp, C.c_int, vp, vp],
        "topt_b200_filter_apply_dev": [vp, vp, C.c_int, vp, vp],
        "topt_b200_csr_apply": [vp, i64, vp, vp, vp, C.c_int, vp, vp],
        "topt_b200_interpolate_stiffness_dev": [vp, i64, i32, vp, d, d, d, vp, vp, vp],
        "topt_b200_element_stiffness_q4": [d, d, vp],
        "topt_b200_compliance_gradient_dev": [vp, i32, i32, d, d, vp, i32, vp, vp, vp],
        "topt_b200_ctx_create_lockstep": [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)],
        "topt_b200_pgd_step_lockstep": [C.c_int, vp, vp, i64, vp, vp, vp, vp, vp],
        "topt_b200_fe_solve_dev": [vp, i32, i32, d, d, vp, vp, i64, vp, vp, i64, d, vp, vp, vp],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = None if name.startswith("topt_b200_default") else C.c_int
    lib.topt_b200_filter_destroy.argtypes = [vp]
    lib.topt_b200_filter_destroy.restype = None
    lib.topt_b200_filter_nnz.argtypes = [vp]
    lib.topt_b200_filter_nnz.restype = C.c_int64
    _lib = lib
    return lib


def _preload_torch_nccl():
    """Make sure the process's NCCL is torch's (loaded with libtorch_cuda)
    before the library resolves NCCL symbols."""
    try:
        import torch  # noqa: F401
    except Exception:
        pass


def nccl_unique_id() -> bytes:
    _preload_torch_nccl()
    buf = (C.c_ubyte * 128)()
    rc = load().topt_b200_nccl_unique_id(buf, 128)
    if rc != OK:
        raise RuntimeError(f"topt_b200_nccl_unique_id failed ({rc}): NCCL not loadable")
    return bytes(buf)


class RowDesc(C.Structure):
    """topt_row_desc: DENSE (0), CONST (1, a_i = value) or CENTROID
    (2, a_i = sign * ((coord_axis(i) + 0.5) - center) / scale)."""
    _fields_ = [("kind", C.c_int32), ("axis", C.c_int32), ("value", C.c_double),
                ("center", C.c_double), ("scale", C.c_double), ("sign", C.c_double)]


class Context:
    """One CUDA device context of the library (stream, plan, workspaces).
    With rank/world/nccl_id it is one rank of a multi-GPU (NCCL) job."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes = None,
                 lockstep: bool = False):
        self.lib = load()
        h = C.c_void_p()
        if lockstep:
            rc = self.lib.topt_b200_ctx_create_lockstep(int(device), int(rank), int(world),
                                                        C.byref(h))
        elif nccl_id is not None:
            _preload_torch_nccl()
            idb = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            rc = self.lib.topt_b200_ctx_create_ranks(int(device), int(rank), int(world), idb,
                                                     C.byref(h))
        else:
            rc = self.lib.topt_b200_ctx_create(int(device), C.byref(h))
        if rc != OK:
            raise RuntimeError(f"topt_b200_ctx_create(device={device}) failed with status {rc} "
                               "(no CUDA device?)")
        self.h = h
        self.device = device
        self.rank, self.world = rank, world
        self.distributed = nccl_id is not None
        self.lockstep = lockstep

    def close(self):
        if self.h:
            self.lib.topt_b200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return self.lib.topt_b200_last_error(self.h).decode()

    @property
    def launches(self) -> int:
        return int(self.lib.topt_b200_kernel_launches(self.h))

    @property
    def stream(self) -> int:
        return int(self.lib.topt_b200_get_stream(self.h) or 0)

    def set_stream(self, stream_ptr: int):
        self.lib.topt_b200_set_stream(self.h, C.c_void_p(stream_ptr))

    @contextlib.contextmanager
    def ordered_with_torch(self):
        """Device-tensor calls: this context's stream waits for the work torch
        has queued on its current stream (the tensors' producers), and torch's
        stream then waits for ours (the consumers of the outputs) -- event
        waits on the device, no host synchronisation.  A no-op when the
        context already runs on torch's current stream (set_stream)."""
        import torch
        cur = torch.cuda.current_stream(self.device)
        mine = self.stream
        if mine == int(cur.cuda_stream):
            yield
            return
        ext = torch.cuda.ExternalStream(mine, device=self.device)
        ext.wait_stream(cur)
        try:
            yield
        finally:
            cur.wait_stream(ext)

    def set_structured_rows(self, rows, grid=None, index_offset: int = 0):
        """Structured constraint rows for the following device steps (None
        clears): a list of RowDesc, one per constraint row."""
        if not rows:
            self.lib.topt_b200_set_structured_rows(self.h, 0, None, None, 0)
            return
        arr = (RowDesc * len(rows))(*rows)
        g = (C.c_int64 * 3)(*[int(v) for v in grid])
        rc = self.lib.topt_b200_set_structured_rows(self.h, len(rows), arr, g, int(index_offset))
        if rc != OK:
            raise RuntimeError(self.last_error())

    PARITY = {"certified": 0, "strict": 1}

    def set_parity(self, mode: str):
        """'certified' (default) or 'strict' (every undecided decision and every
        Newton-stage sum in the reference's sequential order; include/topt_b200.h)."""
        rc = self.lib.topt_b200_set_parity(self.h, self.PARITY[mode])
        if rc != OK:
            raise RuntimeError(self.last_error())

    @property
    def parity(self) -> str:
        v = self.lib.topt_b200_get_parity(self.h)
        return {0: "certified", 1: "strict"}.get(v, str(v))

    def set_profiling(self, on: bool):
        self.lib.topt_b200_set_profiling(self.h, 1 if on else 0)

    def step_time(self):
        """(total_ms, jobs, max_ms) of whole-job device time since the last call
        (profiling on): plan upload -> kernel(s) -> results download."""
        t = C.c_double(0); n = C.c_int64(0); mx = C.c_double(0)
        self.lib.topt_b200_step_time(self.h, C.byref(t), C.byref(n), C.byref(mx))
        return t.value, n.value, mx.value

    def kernel_time(self):
        """(total_ms, launches, max_ms) of profiled pass launches since the last call."""
        t = C.c_double(0); n = C.c_int64(0); mx = C.c_double(0)
        self.lib.topt_b200_kernel_time(self.h, C.byref(t), C.byref(n), C.byref(mx))
        return t.value, n.value, mx.value


_ctx = {}


def context(device: int = 0) -> Context:
    c = _ctx.get(device)
    if c is None:
        c = Context(device)
        _ctx[device] = c
    return c
