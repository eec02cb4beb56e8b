"""Device-side plumbing: the ghosted-slab field layout and the native plan.

Layout (``include/bspde_b200.h``): a field of the local extended grid is a
torch float64 tensor ``buf[nz + 2*ghost, ny, pitch]`` on the GPU, owned plane
``k`` at ``buf[k + ghost]``, ``pitch = nx`` rounded up to even (16-byte rows
for TMA).  Ghost planes (``ghost = degree``) carry neighbour-slab planes in
multi-GPU runs and zeros at physical domain ends.  At 930^3 a field is 6.4 GB.
A heat run keeps u (= x), F, r, Ap (b shares Ap's storage: it is dead once
r0 = b - A x0 is formed) and the ring of R search directions resident:
4 + R fields (``heat_memory_plan``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NativeLibraryError, ValidationError


def _torch():
    import torch

    return torch


def require_cuda(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise NativeLibraryError("the b200 strategy needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    lib = N.load()
    if not lib.bspde_device_ok(dev.index):
        raise NativeLibraryError(f"device {dev} is not an sm_100 (B200-class) GPU")
    return dev


@dataclass(frozen=True)
class SlabLayout:
    nz: int          # owned z planes
    ny: int
    nx: int
    ghost: int
    z_offset: int = 0
    nz_global: int = None

    def __post_init__(self):
        if self.nz_global is None:
            object.__setattr__(self, "nz_global", self.nz)

    @property
    def pitch(self) -> int:
        return self.nx + (self.nx & 1)

    @property
    def buf_shape(self):
        return (self.nz + 2 * self.ghost, self.ny, self.pitch)

    @property
    def owned_shape(self):
        return (self.nz, self.ny, self.nx)

    @property
    def bytes(self) -> int:
        return int(np.prod(self.buf_shape)) * 8

    def alloc(self, device):
        torch = _torch()
        return torch.zeros(self.buf_shape, dtype=torch.float64, device=device)

    def alloc_ring(self, device, n=None):
        """``n`` (default 2) fields back to back: the CG search-direction ring."""
        torch = _torch()
        n = N.RING_DEFAULT if n is None else n
        return torch.zeros((n,) + self.buf_shape, dtype=torch.float64, device=device)

    def owned(self, buf):
        return buf[self.ghost:self.ghost + self.nz, :, :self.nx]

    def upload(self, arr, device, buf=None):
        """Host/torch array of the owned shape -> (new or given) device buffer."""
        torch = _torch()
        if buf is None:
            buf = self.alloc(device)
        src = arr if isinstance(arr, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(arr, dtype=np.float64))
        src = src.reshape(self.owned_shape)
        self.owned(buf).copy_(src, non_blocking=False)
        return buf

    def download(self, buf) -> np.ndarray:
        return self.owned(buf).cpu().numpy().copy()


class NativePlan:
    """Owns one ``bspde_plan`` (operator tables on the device + launch setup)."""

    def __init__(self, data, layout: SlabLayout, device, precond="jacobi"):
        self.data = data
        self.layout = layout
        self.device = device
        self.lib = N.load()
        R = 2 * data.n_b + 1
        self._keep = []

        def arr(a):
            a = np.ascontiguousarray(a, dtype=np.float64).ravel()
            self._keep.append(a)
            return a.ctypes.data_as(N._dptr)

        d = N.PlanDesc()
        d.device = int(device.index)
        d.degree = int(data.n_b)
        d.nz, d.ny, d.nx = layout.nz, layout.ny, layout.nx
        d.nz_global = layout.nz_global
        d.z_offset = layout.z_offset
        for a in range(3):
            d.ew[a] = data.mass[a].ew
            d.mass_table[a] = arr(data.mass[a].table)
            d.stiff_table[a] = arr(data.stiff[a].table)
            assert data.mass[a].table.shape[1] == R
        self.inv_table = data.inv_diag_table(precond)
        d.inv_diag_table = arr(self.inv_table)
        d.pitch_y = layout.pitch
        d.c_mass = float(data.c_mass)
        for a in range(3):
            d.c_stiff[a] = float(data.c_stiff[a])
        h = C.c_void_p()
        N.check(self.lib.bspde_plan_create(C.byref(d), C.byref(h)))
        self.handle = h
        self.desc = d

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            self.lib.bspde_plan_destroy(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.lib.bspde_launch_count(self.handle))

    def scratch(self):
        torch = _torch()
        n = int(self.lib.bspde_scratch_bytes(self.handle))
        return torch.zeros(n, dtype=torch.uint8, device=self.device)

    # thin wrappers ------------------------------------------------------
    def apply(self, c, out, stream=None):
        N.check(self.lib.bspde_apply(self.handle, N.ptr(c), N.ptr(out), N.stream_handle(stream)))

    def mass_apply(self, c, f, cm, a, out, stream=None):
        N.check(self.lib.bspde_mass_apply(self.handle, N.ptr(c), N.ptr(f), float(cm), float(a),
                                          N.ptr(out), N.stream_handle(stream)))

    def jacobi_diagonal(self, out, stream=None):
        tab = np.ascontiguousarray(self.data.diag_table(), dtype=np.float64)
        N.check(self.lib.bspde_jacobi_diagonal(self.handle, tab.ctypes.data_as(N._dptr),
                                               N.ptr(out), N.stream_handle(stream)))

    def pcg(self, b, x, r, pring, ap, scratch, history, tol, max_iter, record_history, has_x0,
            poll_every=8, stream=None):
        cfg = N.CgConfig(float(tol), int(max_iter), int(bool(record_history)),
                         int(bool(has_x0)), int(poll_every), int(pring.shape[0]))
        rep = N.CgReport()
        N.check(self.lib.bspde_pcg_solve(self.handle, N.ptr(b), N.ptr(x), N.ptr(r), N.ptr(pring),
                                         N.ptr(ap), N.ptr(scratch), N.ptr(history),
                                         C.byref(cfg), C.byref(rep), N.stream_handle(stream)))
        return rep

    def heat_step(self, u, f, cm, a, r, pring, ap, scratch, history, tol, max_iter,
                  record_history, poll_every=8, stream=None):
        """One implicit-Euler step in place: (M + dt K) u <- cm M u + a f,
        x0 = u; the RHS is fused into the first residual (bspde_heat_step)."""
        cfg = N.CgConfig(float(tol), int(max_iter), int(bool(record_history)), 1,
                         int(poll_every), int(pring.shape[0]))
        rep = N.CgReport()
        N.check(self.lib.bspde_heat_step(self.handle, N.ptr(u), N.ptr(f), float(cm), float(a),
                                         N.ptr(r), N.ptr(pring), N.ptr(ap), N.ptr(scratch),
                                         N.ptr(history), C.byref(cfg), C.byref(rep),
                                         N.stream_handle(stream)))
        return rep

    def heat_residual(self, u, f, cm, a, r, scratch, fuse, stream=None):
        N.check(self.lib.bspde_heat_residual(self.handle, N.ptr(u), N.ptr(f), float(cm),
                                             float(a), N.ptr(r), N.ptr(scratch), int(fuse),
                                             N.stream_handle(stream)))

    # step-wise CG (multi-GPU driver)
    def cg_setup(self, scratch, history, tol, max_iter, record_history, has_x0, stream=None,
                 p_ring=None):
        cfg = N.CgConfig(float(tol), int(max_iter), int(bool(record_history)),
                         int(bool(has_x0)), 0, int(p_ring or N.RING_DEFAULT))
        N.check(self.lib.bspde_cg_setup(self.handle, N.ptr(scratch), N.ptr(history),
                                        C.byref(cfg), N.stream_handle(stream)))

    def cg_residual(self, b, x, r, scratch, fuse, stream=None):
        N.check(self.lib.bspde_cg_residual(self.handle, N.ptr(b), N.ptr(x), N.ptr(r),
                                           N.ptr(scratch), int(fuse), N.stream_handle(stream)))

    def cg_pass_a(self, x, r, p_in, p_out, ap, scratch, fuse, stream=None):
        """p_k, Ap_k, <p_k, Ap_k> and x += alpha_{k-1} p_{k-1} (k >= 1)."""
        N.check(self.lib.bspde_cg_pass_a(self.handle, N.ptr(x), N.ptr(r), N.ptr(p_in),
                                         N.ptr(p_out), N.ptr(ap), N.ptr(scratch), int(fuse),
                                         N.stream_handle(stream)))

    def cg_pass_a_range(self, x, r, p_in, p_out, ap, scratch, z_begin, z_count, accumulate,
                        fuse=0, stream=None):
        """Pass A on the owned output planes [z_begin, z_begin + z_count)."""
        N.check(self.lib.bspde_cg_pass_a_range(self.handle, N.ptr(x), N.ptr(r), N.ptr(p_in),
                                               N.ptr(p_out), N.ptr(ap), N.ptr(scratch),
                                               int(z_begin), int(z_count), int(bool(accumulate)),
                                               int(fuse), N.stream_handle(stream)))

    def cg_pass_b(self, r, ap, scratch, fuse, stream=None):
        N.check(self.lib.bspde_cg_pass_b(self.handle, N.ptr(r), N.ptr(ap), N.ptr(scratch),
                                         int(fuse), N.stream_handle(stream)))

    def cg_flush_x(self, x, pring, scratch, stream=None):
        N.check(self.lib.bspde_cg_flush_x(self.handle, N.ptr(x), N.ptr(pring), N.ptr(scratch),
                                          N.stream_handle(stream)))

    def cg_finalize(self, scratch, kind, stream=None):
        N.check(self.lib.bspde_cg_finalize(self.handle, N.ptr(scratch), int(kind),
                                           N.stream_handle(stream)))

    def cg_finalize_gathered(self, scratch, gathered, world, kind, stream=None):
        N.check(self.lib.bspde_cg_finalize_gathered(self.handle, N.ptr(scratch), N.ptr(gathered),
                                                    int(world), int(kind),
                                                    N.stream_handle(stream)))

    def set_peers(self, peers):
        """z-slab peer halos (``_native.SlabPeers`` or None to clear)."""
        N.check(self.lib.bspde_slab_set_peers(self.handle,
                                              C.byref(peers) if peers is not None else None))

    def cg_read(self, scratch, stream=None):
        rep = N.CgReport()
        active = C.c_int32()
        N.check(self.lib.bspde_cg_read_report(self.handle, N.ptr(scratch), C.byref(rep),
                                              C.byref(active), N.stream_handle(stream)))
        return rep, bool(active.value)


# resident fields of a heat run besides the p ring: u (= x), F, r, Ap (= b)
HEAT_BASE_FIELDS = 4
HBM_BUDGET = 175e9  # bytes of HBM3e a rank may fill with fields (B200: 180 GB usable)


def ipc_export(t):
    """CUDA IPC handle (64 bytes) and byte offset of a device tensor's data."""
    lib = N.load()
    h = (C.c_char * 64)()
    off = C.c_uint64()
    N.check(lib.bspde_ipc_export(N.ptr(t), h, C.byref(off)))
    return bytes(h), int(off.value)


def ipc_import(handle, offset):
    """Map another process's allocation (``ipc_export``): a device pointer."""
    lib = N.load()
    out = C.c_void_p()
    N.check(lib.bspde_ipc_import(C.create_string_buffer(bytes(handle), 64), int(offset),
                                 C.byref(out)))
    return int(out.value)


def ipc_close(ptr):
    N.check(N.load().bspde_ipc_close(C.c_void_p(ptr)))


def heat_memory_plan(cext, degree, world=1, budget=HBM_BUDGET, ring=None):
    """Per-rank resident bytes of a heat run on ``world`` z-slabs.

    Fields: u, F, r, Ap (b aliases Ap) and the search-direction ring (R = 2:
    p_{k-1}, p_k; pass A applies the x updates).  Returns dict(ring,
    fields, field_bytes, bytes).  1536^3 p=3 on one GPU: 6 fields x 29.1 GB =
    174.7 GB."""
    from .errors import ConfigurationError

    nzg, ny, nx = (int(v) for v in cext)
    nz = -(-nzg // int(world))  # the largest slab
    field = SlabLayout(nz, ny, nx, ghost=int(degree)).bytes
    for R in ((ring,) if ring else (N.RING_DEFAULT,)):
        total = (HEAT_BASE_FIELDS + R) * field
        if total <= budget:
            return dict(ring=R, fields=HEAT_BASE_FIELDS + R, field_bytes=field, bytes=total)
    raise ConfigurationError(
        f"{cext} (degree {degree}) on {world} rank(s) needs {(HEAT_BASE_FIELDS + 2) * field / 1e9:.1f}"
        f" GB per rank > {budget / 1e9:.0f} GB; use more GPUs")


def choose_ring(layout=None, device=None):
    """Ring length of a CG work set: 2 (p_{k-1}, p_k; pass A applies x += alpha
    p, so no longer ring is needed).  ``BSPDE_P_RING_LEN`` = 4 keeps four
    fields (testing the ring indexing)."""
    import os

    env = os.environ.get("BSPDE_P_RING_LEN")
    if env:
        R = int(env)
        if R not in (2, N.P_RING):
            raise ValidationError(f"BSPDE_P_RING_LEN must be 2 or {N.P_RING}, got {env}")
        return R
    return N.RING_DEFAULT


def check_host_field(c, shape, what="input coefficients"):
    c = np.asarray(c)
    if c.shape != tuple(shape):
        raise ValidationError(f"extents {c.shape} != operator grid {tuple(shape)}")
    if not np.all(np.isfinite(c)):
        raise ValidationError(f"{what} contain non-finite values")
    return np.ascontiguousarray(c, dtype=np.float64)
