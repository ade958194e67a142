"""ctypes binding of the C-ABI in include/pintmk_b200.h.

The shared library ``libpmk_b200.so`` (hand-written sm_100a kernels plus the
native FGMRES recursion) is built in-tree by ``build()`` (nvcc through the
Makefile in ``csrc/``).  There is no fallback: if the library is missing or
no CUDA device is present, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int32, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# PMK_LIB overrides the library path (tuning builds, e.g. libpmk_b200_<variant>.so)
LIB_PATH = os.environ.get("PMK_LIB") or os.path.join(_HERE, "libpmk_b200.so")
CSRC = os.path.join(_HERE, "csrc")

PMK_ERR_ARG = 1001
PMK_ERR_SHAPE = 1002
PMK_ERR_UNSUPPORTED = 1003
PMK_ERR_STATE = 1004
PMK_COARSE_DST = 1
PMK_COARSE_DENSE = 2
PMK_COARSE_EIG = 3
PMK_COARSE_PCR = 4
PMK_COARSE_LINE = 5


class Stencil(ctypes.Structure):
    _fields_ = [("var", c_int32), ("c", c_double * 5), ("coef", c_void_p)]


class LevelDesc(ctypes.Structure):
    _fields_ = [("dim", c_int32), ("nx", c_int32), ("ny", c_int32),
                ("n_steps", c_int32), ("diag_t", Stencil), ("sub_t", Stencil),
                ("dropped", c_void_p)]


class PairDesc(ctypes.Structure):
    _fields_ = [("nu", c_int32), ("n_T", c_int32), ("m_fine", c_int32),
                ("m_coarse", c_int32), ("group_of", c_void_p), ("y_ptr", c_void_p),
                ("y_idx", c_void_p), ("y_val", c_void_p), ("mgrit", c_int32),
                ("dim", c_int32), ("nx", c_int32), ("ny", c_int32), ("sx", c_void_p),
                ("sy", c_void_p), ("fft_x", c_void_p), ("fft_y", c_void_p),
                ("fft_scale", c_double), ("ratio", c_void_p), ("work0", c_void_p),
                ("work1", c_void_p), ("work2", c_void_p), ("coarse_out", c_void_p),
                ("z_ptr", c_void_p), ("z_idx", c_void_p), ("z_val", c_void_p)]


class CoarseDesc(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("dim", c_int32), ("nx", c_int32), ("ny", c_int32),
                ("n_steps", c_int32), ("dropped", c_void_p), ("sx", c_void_p),
                ("sy", c_void_p), ("delta", c_void_p), ("beta", c_void_p),
                ("dinv", c_void_p), ("coupling", Stencil), ("work0", c_void_p),
                ("work1", c_void_p), ("fft_x", c_void_p), ("fft_y", c_void_p),
                ("fft_scale", c_double), ("ix", c_void_p), ("iy", c_void_p),
                ("n_cx", c_int32), ("n_cy", c_int32), ("cx_h", c_void_p), ("cx_u", c_void_p),
                ("cy_h", c_void_p), ("cy_u", c_void_p), ("coupling_b", c_double),
                ("seg_start", c_void_p), ("n_seg", c_int32), ("pcr_levels", c_int32),
                ("pcr_alpha", c_void_p), ("pcr_gamma", c_void_p), ("pcr_inv", c_void_p),
                ("line_g", c_void_p), ("line_l", c_void_p), ("line_u", c_void_p),
                ("line_cs", c_int32)]


# name -> (restype, argtypes); exactly the functions include/pintmk_b200.h declares
SIGNATURES = {
    "pmk_version": (ctypes.c_char_p, []),
    "pmk_stmv": (c_int32, [POINTER(LevelDesc), c_void_p, c_void_p, c_void_p]),
    "pmk_restrict": (c_int32, [POINTER(PairDesc), c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmk_interpolate": (c_int32, [POINTER(PairDesc), c_void_p, c_void_p, c_void_p]),
    "pmk_stmv_shift_restrict": (c_int32, [POINTER(LevelDesc), POINTER(PairDesc), c_double,
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmk_interp_sub_stmv": (c_int32, [POINTER(LevelDesc), POINTER(PairDesc), c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmk_coarsest_solve": (c_int32, [POINTER(CoarseDesc), c_void_p, c_void_p, c_void_p]),
    "pmk_dot": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "pmk_nrm2": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p]),
    "pmk_residual_nrm2": (c_int32, [POINTER(LevelDesc), c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p]),
    "pmk_residual": (c_int32, [POINTER(LevelDesc), c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p]),
    "pmk_axpy": (c_int32, [c_double, c_void_p, c_void_p, c_int64, c_void_p]),
    "pmk_hier_create": (c_void_p, [c_int32, c_double]),
    "pmk_hier_destroy": (None, [c_void_p]),
    "pmk_hier_set_level": (c_int32, [c_void_p, c_int32, POINTER(LevelDesc),
                                     POINTER(PairDesc), c_int32]),
    "pmk_hier_set_coarse": (c_int32, [c_void_p, POINTER(CoarseDesc)]),
    "pmk_hier_set_buffers": (c_int32, [c_void_p, c_int32, c_void_p, POINTER(c_void_p),
                                       POINTER(c_void_p), c_int32, c_void_p, c_void_p]),
    "pmk_fgmres_begin": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_double, c_void_p]),
    "pmk_fgmres_step": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "pmk_fgmres_finish": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p]),
    "pmk_fgmres_finish_rows": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_int32,
                                         c_void_p]),
    "pmk_fgmres_state": (c_int32, [c_void_p, c_int32, POINTER(c_double), POINTER(c_double),
                                   POINTER(c_double), POINTER(c_double), POINTER(c_int32),
                                   c_void_p]),
    "pmk_fgmres_fixed": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p]),
    "pmk_apply_preconditioner": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p,
                                           c_void_p]),
    "pmk_profile_begin": (c_int32, [c_int32]),
    "pmk_profile_end": (c_int32, [POINTER(c_double), c_int32, POINTER(c_int32)]),
    "pmk_profile_end_levels": (c_int32, [POINTER(c_double), c_int32, POINTER(c_int32)]),
    "pmk_profile_category": (ctypes.c_char_p, [c_int32]),
    "pmk_launch_count": (c_int64, []),
    "pmk_lazy_basis": (c_int32, []),
    "pmk_fgmres_snapshot": (c_int32, [c_void_p, c_int32, c_int32, c_void_p]),
    "pmk_fgmres_snapshot_read": (c_int32, [c_void_p, c_int32, c_int32, c_void_p]),
    "pmk_div_check": (c_int32, [c_void_p, c_double, c_int64, c_void_p, c_void_p]),
    "pmk_dgemm": (c_int32, [c_int32, c_int32, c_int32, c_void_p, c_int32, c_int64, c_void_p,
                            c_int32, c_int64, c_void_p, c_int32, c_int64, c_int32, c_void_p]),
}

_lib = None


def build(force: bool = False, quiet: bool = True) -> str:
    """Compile libpmk_b200.so for sm_100a in-tree (nvcc via csrc/Makefile)."""
    if force:
        subprocess.run(["make", "-C", CSRC, "clean"], check=True,
                       capture_output=quiet)
    proc = subprocess.run(["make", "-C", CSRC, "-j4"], capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"building libpmk_b200.so failed:\n{proc.stdout}\n{proc.stderr}")
    return LIB_PATH


def load():
    """Load the shared library (building it first if absent); raise if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class PmkError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc in (PMK_ERR_ARG, PMK_ERR_SHAPE):
        raise ValueError(f"{what}: invalid argument (code {rc})")
    if rc == PMK_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: unsupported configuration")
    if rc == PMK_ERR_STATE:
        raise PmkError(f"{what}: call order violated")
    raise PmkError(f"{what}: CUDA error {rc}")


def require_cuda():
    """The product path has no CPU fallback: fail loudly without a GPU."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2401_00228_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    load()
    return torch


def stream_ptr():
    import torch

    return c_void_p(torch.cuda.current_stream().cuda_stream)


def profile_begin(with_events: bool = True) -> None:
    check(load().pmk_profile_begin(1 if with_events else 0), "profile_begin")


def profile_end() -> dict:
    """{category: {launches, ms, bytes, flops}} since profile_begin (synchronises)."""
    lib = load()
    stats = (c_double * 64)()
    n = c_int32(0)
    check(lib.pmk_profile_end(stats, 16, ctypes.byref(n)), "profile_end")
    out = {}
    for c in range(n.value):
        name = lib.pmk_profile_category(c).decode()
        launches, ms, nbytes, flops = stats[4 * c: 4 * c + 4]
        if launches:
            out[name] = {"launches": int(launches), "ms": ms, "bytes": nbytes, "flops": flops}
    return out


HINTS = {-1: None, 1: "restriction", 2: "interpolation"}


def profile_end_levels() -> list[dict]:
    """Records since profile_begin split by attribution: a list of
    {level, hint, category, launches, ms, bytes, flops} (synchronises)."""
    lib = load()
    cap = 512
    rows = (c_double * (7 * cap))()
    n = c_int32(0)
    check(lib.pmk_profile_end_levels(rows, cap, ctypes.byref(n)), "profile_end_levels")
    out = []
    for i in range(n.value):
        lvl, hint, cat, launches, ms, nbytes, flops = rows[7 * i: 7 * i + 7]
        out.append({"level": int(lvl), "hint": HINTS.get(int(hint)),
                    "category": lib.pmk_profile_category(int(cat)).decode(),
                    "launches": int(launches), "ms": ms, "bytes": nbytes, "flops": flops})
    return out


def launch_count() -> int:
    return int(load().pmk_launch_count())


def ptr(t) -> c_void_p:
    return c_void_p(0 if t is None else t.data_ptr())


def lazy_basis() -> bool:
    """True when the native solver keeps a lazy (raw) Krylov basis."""
    return bool(load().pmk_lazy_basis())
