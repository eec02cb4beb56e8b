"""ctypes binding of the sm_100a C ABI (``include/bspde_b200.h``).

This is the only door to the hot path.  There is no CPU fallback: if the
library is missing or a call fails, :class:`NativeLibraryError` is raised.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NativeLibraryError

HERE = os.path.dirname(os.path.abspath(__file__))
# BSPDE_LIB selects a tuning variant built by build.py --out=... (development
# only; the variant is the same source with different -D constants).
LIB_PATH = os.environ.get("BSPDE_LIB") or os.path.join(HERE, "libbspde_b200.so")

P_RING = 4  # BSPDE_P_RING: the longest search-direction ring (include/bspde_b200.h)
RING_DEFAULT = 2  # pass A applies x, so two fields (p_{k-1}, p_k) suffice

BSPDE_CG_RUNNING = 0
BSPDE_CG_CONVERGED = 1
BSPDE_CG_MAXITER = 2
BSPDE_CG_INDEFINITE = 3
BSPDE_CG_DIVERGED = 4
BSPDE_CG_ZERO_RHS = 5

_dptr = C.POINTER(C.c_double)


class PlanDesc(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("degree", C.c_int32),
        ("nz", C.c_int32), ("ny", C.c_int32), ("nx", C.c_int32),
        ("nz_global", C.c_int32),
        ("z_offset", C.c_int32),
        ("ew", C.c_int32 * 3),
        ("pitch_y", C.c_int64),
        ("mass_table", _dptr * 3),
        ("stiff_table", _dptr * 3),
        ("inv_diag_table", _dptr),
        ("c_mass", C.c_double),
        ("c_stiff", C.c_double * 3),
    ]


class CgConfig(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_int32),
        ("record_history", C.c_int32),
        ("has_x0", C.c_int32),
        ("poll_every", C.c_int32),
        ("p_ring", C.c_int32),
    ]


class StencilDesc(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("degree", C.c_int32),
        ("param_degree", C.c_int32),
        ("nz", C.c_int32), ("ny", C.c_int32), ("nx", C.c_int32),
        ("pz", C.c_int32), ("py", C.c_int32), ("px", C.c_int32),
        ("ext", C.c_int32), ("ext_p", C.c_int32),
        ("ew", C.c_int32 * 3),
        ("tables", (_dptr * 2) * 3),
        ("scale_stiff", C.c_double * 3),
        ("scale_mass", C.c_double),
        ("nfaces", C.c_int32),
        ("face_axis", C.c_int32 * 6),
        ("face_side", C.c_int32 * 6),
        ("face_weight", C.c_double * 6),
        ("face_values", _dptr),
        ("mass_gram", _dptr),
        ("step", C.c_double * 3),
        ("degenerate", C.c_int32 * 3),
    ]


class MaskDesc(C.Structure):
    _fields_ = [
        ("occupancy", C.c_void_p),
        ("cells", C.c_int32 * 3),
        ("node_class", C.c_void_p),
        ("brows", C.c_void_p),
        ("nbrows", C.c_int64),
        ("brows_k", C.c_void_p),
        ("jlo", C.c_int32), ("nj", C.c_int32),
        ("blo", C.c_int32), ("nbp", C.c_int32),
        ("cell_tri", C.c_void_p),
        ("cell_bil", C.c_void_p),
        ("cell_single", C.c_void_p),
        ("face_vals", C.c_void_p),
        ("fc", C.c_int32),
        ("has_surface", C.c_int32),
        ("surface_weight", C.c_double),
        ("degenerate", C.c_int32 * 3),
    ]


class CgReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("status", C.c_int32),
        ("relative_residual", C.c_double),
        ("residual", C.c_double),
        ("residual0", C.c_double),
        ("rhs_norm", C.c_double),
        ("last_pAp", C.c_double),
    ]


class SlabPeers(C.Structure):
    _fields_ = [
        ("ring", C.c_void_p),
        ("r", C.c_void_p),
        ("ring_stride", C.c_int64),
        ("ring_len", C.c_int32),
        ("lo_nz", C.c_int32),
        ("lo_ring", C.c_void_p),
        ("lo_ring_stride", C.c_int64),
        ("lo_r", C.c_void_p),
        ("hi_ring", C.c_void_p),
        ("hi_ring_stride", C.c_int64),
        ("hi_r", C.c_void_p),
    ]


# (name, restype, argtypes) -- must cover every function in include/bspde_b200.h
_VP = C.c_void_p
SIGNATURES = [
    ("bspde_last_error", C.c_char_p, []),
    ("bspde_version", C.c_int, []),
    ("bspde_device_ok", C.c_int, [C.c_int]),
    ("bspde_plan_create", C.c_int, [C.POINTER(PlanDesc), C.POINTER(_VP)]),
    ("bspde_plan_destroy", C.c_int, [_VP]),
    ("bspde_scratch_bytes", C.c_int64, [_VP]),
    ("bspde_launch_count", C.c_int64, [_VP]),
    ("bspde_apply", C.c_int, [_VP, _VP, _VP, _VP]),
    ("bspde_mass_apply", C.c_int, [_VP, _VP, _VP, C.c_double, C.c_double, _VP, _VP]),
    ("bspde_jacobi_diagonal", C.c_int, [_VP, _dptr, _VP, _VP]),
    ("bspde_pcg_solve", C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                  C.POINTER(CgConfig), C.POINTER(CgReport), _VP]),
    ("bspde_heat_step", C.c_int, [_VP, _VP, _VP, C.c_double, C.c_double, _VP, _VP, _VP, _VP,
                                  _VP, C.POINTER(CgConfig), C.POINTER(CgReport), _VP]),
    ("bspde_heat_residual", C.c_int, [_VP, _VP, _VP, C.c_double, C.c_double, _VP, _VP, C.c_int,
                                      _VP]),
    ("bspde_cg_setup", C.c_int, [_VP, _VP, _VP, C.POINTER(CgConfig), _VP]),
    ("bspde_cg_residual", C.c_int, [_VP, _VP, _VP, _VP, _VP, C.c_int, _VP]),
    ("bspde_cg_pass_a", C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int, _VP]),
    ("bspde_cg_pass_a_range", C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int, C.c_int,
                                        C.c_int, C.c_int, _VP]),
    ("bspde_cg_pass_b", C.c_int, [_VP, _VP, _VP, _VP, C.c_int, _VP]),
    ("bspde_cg_flush_x", C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("bspde_stencil_create", C.c_int, [C.POINTER(StencilDesc), C.POINTER(C.c_void_p)]),
    ("bspde_stencil_destroy", C.c_int, [_VP]),
    ("bspde_stencil_entries", C.c_int64, [_VP]),
    ("bspde_stencil_set_rows", C.c_int, [_VP, _VP, C.c_int64]),
    ("bspde_otf_supported", C.c_int, [_VP]),
    ("bspde_otf_prepare", C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("bspde_otf_apply", C.c_int, [_VP, _VP, _VP, _VP]),
    ("bspde_otf_pcg", C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, C.POINTER(CgConfig),
                                C.POINTER(CgReport), C.c_int32, _VP]),
    ("bspde_stencil_launch_count", C.c_int64, [_VP]),
    ("bspde_stencil_assemble", C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("bspde_stencil_apply", C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("bspde_stencil_diagonal", C.c_int, [_VP, _VP, _VP, _VP]),
    ("bspde_stencil_pcg", C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                    C.POINTER(CgConfig), C.POINTER(CgReport), C.c_int32, _VP]),
    ("bspde_stencil_mask_patch", C.c_int, [_VP, C.POINTER(MaskDesc), _VP, _VP, _VP, _VP]),
    ("bspde_stencil_mask_surface_rhs", C.c_int, [_VP, C.POINTER(MaskDesc), C.c_double, _VP, _VP]),
    ("bspde_resample_axis", C.c_int, [_VP, _VP, _VP, _VP, _VP, C.c_int32, _VP, _VP, C.c_int32,
                                      _VP]),
    ("bspde_banded_solve_lines", C.c_int, [_VP, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                           C.c_int64, C.c_int64, _VP, _VP, C.c_int32, _VP]),
    ("bspde_eval_points", C.c_int, [_VP, _VP, C.c_int64, C.c_int32, _VP, _VP, _VP, _VP]),
    ("bspde_prefilter_lines", C.c_int, [_VP, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                        C.c_int64, C.c_int64, _VP, C.c_int32, C.c_double,
                                        C.c_int32, _VP]),
    ("bspde_reflect_pad", C.c_int, [_VP, _VP, _VP, C.c_int32, C.c_int32, _VP]),
    ("bspde_fir_axis", C.c_int, [_VP, _VP, _VP, _VP, _VP, C.c_int32, C.c_int32, _VP,
                                 C.c_int32, _VP]),
    ("bspde_cg_finalize", C.c_int, [_VP, _VP, C.c_int, _VP]),
    ("bspde_cg_finalize_gathered", C.c_int, [_VP, _VP, _VP, C.c_int, C.c_int, _VP]),
    ("bspde_slab_set_peers", C.c_int, [_VP, C.POINTER(SlabPeers)]),
    ("bspde_ipc_export", C.c_int, [_VP, _VP, C.POINTER(C.c_uint64)]),
    ("bspde_ipc_import", C.c_int, [_VP, C.c_uint64, C.POINTER(_VP)]),
    ("bspde_ipc_close", C.c_int, [_VP]),
    ("bspde_cg_read_report", C.c_int, [_VP, _VP, C.POINTER(CgReport),
                                       C.POINTER(C.c_int32), _VP]),
]

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the native library (once).  Raises NativeLibraryError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"native library {path} not built; run "
                "`python -m paper_1904_03057_b200.build` (no CPU fallback exists)")
        try:
            lib = C.CDLL(path)
        except OSError as e:  # pragma: no cover - environment specific
            raise NativeLibraryError(f"cannot load {path}: {e}") from e
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int):
    if rc != 0:
        msg = load().bspde_last_error()
        raise NativeLibraryError(
            f"bspde native call failed (code {rc}): {msg.decode() if msg else ''}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def ptr(t) -> C.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())


def stream_handle(stream=None) -> C.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
