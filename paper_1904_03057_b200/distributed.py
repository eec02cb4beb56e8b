"""Multi-GPU z-slab execution: one process per GPU, NCCL over NVLink/NVSwitch.

The global extended grid is split along axis 0 ("z", the slowest axis) into
contiguous slabs, one per rank (``SlabPartition``).  Each rank stores its
slab in the ghosted layout of ``device.SlabLayout`` with ``ghost = p`` planes
per side; the kernels read ghosts and write only owned planes.

Per CG iteration (``distributed_pcg``):

  1. halo exchange of r and p_{k-1}: the first/last p owned planes go to the
     lower/upper neighbour's ghost planes (contiguous memory: one send + one
     recv per side and buffer, both buffers in one
     ``torch.distributed.batch_isend_irecv`` group over NCCL);
     p_k's exchange is posted right after the pass A that writes it and
     runs (on the halo communicator's own NCCL stream) under the all-reduce,
     finalize and pass B; r's follows pass B ("pipeline", the default; see
     ``_halo_mode`` for "split", which also runs pass A's interior planes
     under r's exchange through ``bspde_cg_pass_a_range``);
  2. pass A (fuse=0) forms p_k (stored into the ping-pong partner buffer),
     applies x += alpha_{k-1} p_{k-1} on the owned planes and writes the
     local <p, Ap> as a double-double pair; ``all_gather`` of the ranks'
     pairs (64 bytes each); the 1-thread finalize kernel adds them in rank
     order, rounds once and runs the scalar update on every rank;
  3. pass B (fuse=0): r -= alpha Ap, local <r, D^-1 r>, <r, r>; all-gather;
     finalize.

The rounded scalars equal the single-device ones (both are the correctly
rounded dot products, bspde_b200.cu "Double-double"), so an N-rank solve
takes the same iterations as one GPU, bit for bit.

Every rank holds identical scalar state, so the device-side ``active`` flag
(stop rule, guards) agrees everywhere; the host polls it every
``poll_every`` iterations.  Iterations after convergence are no-ops.  There
is no collective on the data path other than the halo planes and the scalar
sums.

Transport: NCCL over NVLink/NVSwitch in production (one process per GPU).
With the gloo backend (several ranks sharing one GPU in the multi-process
GPU test, or CPU runs) the halo planes and the scalar sums of CUDA tensors
are staged through host memory (``HaloExchanger`` / ``_all_gather_fn``).

The orchestration is written against a small ops interface so it can be
exercised on CPU with the gloo backend (tests/test_distributed_cpu.py); the
product implementation is ``NativeSlabOps`` (the sm_100a kernels).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ConfigurationError, ValidationError
from .solver import SolveConfig, report_from


@dataclass(frozen=True)
class SlabPartition:
    """Balanced split of ``nz_global`` planes over ``world`` ranks."""

    nz_global: int
    world: int
    rank: int

    def __post_init__(self):
        if not 0 <= self.rank < self.world:
            raise ValidationError(f"rank {self.rank} not in [0, {self.world})")
        if self.nz_global < self.world:
            raise ConfigurationError(
                f"{self.nz_global} z planes cannot be split over {self.world} ranks")

    def bounds(self, rank=None):
        r = self.rank if rank is None else rank
        base, extra = divmod(self.nz_global, self.world)
        lo = r * base + min(r, extra)
        return lo, lo + base + (1 if r < extra else 0)

    @property
    def z_offset(self):
        return self.bounds()[0]

    @property
    def nz(self):
        lo, hi = self.bounds()
        return hi - lo

    def check_min(self, planes):
        for r in range(self.world):
            lo, hi = self.bounds(r)
            if hi - lo < planes:
                raise ConfigurationError(
                    f"rank {r} owns {hi - lo} z planes < {planes} (degree); use fewer ranks")


def _torch():
    import torch

    return torch


class HaloExchanger:
    """Fills the ghost planes of a slab buffer from the neighbouring ranks."""

    def __init__(self, layout, rank, world, group=None):
        self.layout = layout
        self.rank = rank
        self.world = world
        self.group = group

    def __call__(self, *bufs):
        """Exchange the ghost planes of every buffer in ``bufs`` in ONE
        batched P2P group (the CG loop passes r and p_{k-1} together, so an
        iteration pays one group launch / NVLink round trip, not two)."""
        self.wait(self.start(*bufs))

    @staticmethod
    def wait(works):
        """Complete a started exchange (NCCL: the current stream waits on the
        transfer; gloo: the host blocks)."""
        for req in works:
            req.wait()

    def _staged(self, buf):
        import torch.distributed as dist

        return buf.is_cuda and dist.get_backend(self.group) == "gloo"

    def start(self, *bufs):
        """Post the exchange and return its work handles without waiting, so
        kernels that read no ghost plane can run while it is in flight."""
        if self.world == 1:
            return []
        import torch.distributed as dist

        if bufs and self._staged(bufs[0]):
            return self._start_staged(bufs)
        g, nz = self.layout.ghost, self.layout.nz
        ops = []
        for buf in bufs:
            if self.rank > 0:  # lower neighbour: my first g planes <-> its top ghosts
                ops.append(dist.P2POp(dist.isend, buf[g:2 * g], self.rank - 1, self.group))
                ops.append(dist.P2POp(dist.irecv, buf[0:g], self.rank - 1, self.group))
            if self.rank < self.world - 1:  # upper neighbour
                ops.append(dist.P2POp(dist.isend, buf[nz:nz + g], self.rank + 1, self.group))
                ops.append(dist.P2POp(dist.irecv, buf[nz + g:nz + 2 * g], self.rank + 1,
                                      self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def _start_staged(self, bufs):
        """gloo + CUDA tensors: copy the boundary planes to the host, exchange
        them with gloo P2P and copy the received planes into the ghost planes
        (synchronous; the returned handle list is empty)."""
        import torch.distributed as dist

        g, nz = self.layout.ghost, self.layout.nz
        for buf in bufs:
            ops, recvs = [], []
            if self.rank > 0:
                lo = buf[g:2 * g].cpu()
                rlo = lo.new_empty(lo.shape)
                ops += [dist.P2POp(dist.isend, lo, self.rank - 1, self.group),
                        dist.P2POp(dist.irecv, rlo, self.rank - 1, self.group)]
                recvs.append((slice(0, g), rlo))
            if self.rank < self.world - 1:
                hi = buf[nz:nz + g].cpu()
                rhi = hi.new_empty(hi.shape)
                ops += [dist.P2POp(dist.isend, hi, self.rank + 1, self.group),
                        dist.P2POp(dist.irecv, rhi, self.rank + 1, self.group)]
                recvs.append((slice(nz + g, nz + 2 * g), rhi))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for sl, t in recvs:
                buf[sl].copy_(t)
        return []


def _all_gather_fn(world, group=None):
    """t (k values) -> the rank-major (world x k) gather, on t's device."""
    import torch.distributed as dist

    torch = _torch()

    def fn(t, out):
        if t.is_cuda and dist.get_backend(group) == "gloo":  # host-staged (see module doc)
            parts = [torch.empty_like(t, device="cpu") for _ in range(world)]
            dist.all_gather(parts, t.cpu(), group=group)
            out.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(out, t, group=group)

    return fn


class NativeSlabOps:
    """Step-wise CG through the C ABI on one rank's slab (fuse = 0).

    The passes leave this rank's dot products as double-double pairs (the
    first 64 bytes of scratch); ``reduce`` all-gathers the world's pairs (8
    doubles per rank) and the finalize kernel adds them in rank order before
    rounding once, so the scalars -- and the iterates -- are bit-identical on
    every rank and to the single-device solve."""

    def __init__(self, plan, world=1, group=None, peers=None):
        self.plan = plan
        self.world = world
        self._gather = _all_gather_fn(world, group) if world > 1 else None
        self._gathered = None
        self.peers = peers  # _native.SlabPeers of this rank's work set, or None
        self.peer_ready = peers is not None

    def use_peers(self, on):
        """Pass B stores the boundary planes of r and p_k into the
        neighbours' ghost planes itself (bspde_slab_set_peers)."""
        self.plan.set_peers(self.peers if on else None)

    def reduce(self, scratch, n, kind):
        """Cross-rank scalar step after a fuse = 0 pass (n sums, finalize kind)."""
        if self.world == 1:
            self.plan.cg_finalize(scratch, kind)
            return
        torch = _torch()
        if self._gathered is None or self._gathered.device != scratch.device:
            self._gathered = torch.empty(self.world * 8, dtype=torch.float64, device=scratch.device)
        self._gather(scratch[:64].view(torch.float64), self._gathered)
        self.plan.cg_finalize_gathered(scratch, self._gathered, self.world, kind)

    def setup(self, scratch, history, cfg, has_x0, ring=None):
        self.plan.cg_setup(scratch, history, cfg.tol, cfg.max_iter, cfg.record_history, has_x0,
                           p_ring=ring)

    def residual(self, b, x, r, scratch):
        self.plan.cg_residual(b, x, r, scratch, 0)

    def heat_residual(self, u, F, cm, a, r, scratch):
        """r0 = (cm M u + a F) - A u and the three initial sums, b never formed."""
        self.plan.heat_residual(u, F, cm, a, r, scratch, 0)

    def pass_a(self, x, r, p_in, p_out, ap, scratch):
        self.plan.cg_pass_a(x, r, p_in, p_out, ap, scratch, 0)

    def pass_a_range(self, x, r, p_in, p_out, ap, scratch, z_begin, z_count, accumulate):
        self.plan.cg_pass_a_range(x, r, p_in, p_out, ap, scratch, z_begin, z_count, accumulate, 0)

    def pass_b(self, r, ap, scratch):
        self.plan.cg_pass_b(r, ap, scratch, 0)

    def flush_x(self, x, pring, scratch):
        self.plan.cg_flush_x(x, pring, scratch)

    def read(self, scratch):
        return self.plan.cg_read(scratch)


HALO_MODES = ("peer", "pipeline", "split", "off")


def _halo_mode(ops, halo):
    """``BSPDE_HALO_OVERLAP``: "peer" (default when the neighbours' fields are
    mapped), "pipeline" (default otherwise), "split" or "off" ("0").

    * peer -- the kernels store the halo planes themselves: pass B writes
      the new r and the preceding pass A's p_k of its first / last p owned
      planes into the neighbours' ghost planes (NVLink peer memory, mapped
      by CUDA IPC); the scalar all-gather after pass B orders those stores
      before the neighbours' next pass A, so no halo transfer is issued per
      iteration;

    * pipeline -- p_k's ghost planes travel while the <p,Ap> all-reduce,
      finalize and pass B of the same iteration run (the exchange is posted
      right after pass A on the halo communicator, a separate NCCL stream);
      only r's exchange sits between pass B and the next pass A;
    * split -- pipeline, plus pass A split around r's exchange: the interior
      output planes [g, nz - g), which read no ghost plane, run while it is in
      flight, the two g-plane boundary ranges after it lands (costs 2 x 2p
      warm-up planes per tile; tools/time_slab_split.py);
    * off -- both exchanges before pass A.
    """
    if halo.world == 1:
        return "off"
    peer_ready = getattr(ops, "peer_ready", False)
    mode = os.environ.get("BSPDE_HALO_OVERLAP", "peer" if peer_ready else "pipeline")
    mode = "off" if mode == "0" else mode
    if mode not in HALO_MODES:
        raise ConfigurationError(f"BSPDE_HALO_OVERLAP must be one of {HALO_MODES}, got {mode!r}")
    if mode == "peer" and not peer_ready:
        mode = "pipeline"  # the neighbours' fields are not mapped (BSPDE_PEER_HALO=0 / no IPC)
    lay = halo.layout
    if mode == "split" and not (hasattr(ops, "pass_a_range") and lay.nz > 2 * lay.ghost):
        mode = "pipeline"  # no interior range on this slab
    return mode


def distributed_pcg(ops, halo, b, x, r, pring, ap, scratch, config: SolveConfig,
                    has_x0=True, history=None, heat=None):
    """Jacobi-PCG over z-slabs (same recurrence and stop rule as solver.pcg);
    ``pring`` holds the ring of search directions (leading axis).  Iteration
    k needs the ghost planes of r_k and p_{k-1}; how their exchange overlaps
    the kernels is ``_halo_mode``."""
    t0 = time.perf_counter()
    mode = _halo_mode(ops, halo)
    g, nz = halo.layout.ghost, halo.layout.nz
    if not has_x0:
        x.zero_()
    R = pring.shape[0]
    ops.setup(scratch, history, config, has_x0, ring=R)
    if hasattr(ops, "use_peers"):
        ops.use_peers(mode == "peer")
    halo(x)
    if heat is not None:  # heat step: b = cm M u + a F fused into the first residual
        F, cm, a = heat
        ops.heat_residual(x, F, cm, a, r, scratch)
    else:
        ops.residual(b, x, r, scratch)
    ops.reduce(scratch, 3, 0)
    if mode == "peer":
        halo(r)  # r_0's ghost planes; from here on pass B stores the halos
    rep, active = ops.read(scratch)
    K = max(1, int(config.poll_every))
    k = 0
    pending_p = []  # the in-flight exchange of p_{k-1} (pipeline / split)
    try:
        while active:
            for _ in range(K):
                # iteration 0 has beta = 0: r itself stands in for p_{-1}
                # (p_0 = D^-1 r + 0 * r; no zeroed field, nothing extra to exchange)
                p_in, p_out = (r if k == 0 else pring[(k - 1) % R]), pring[k % R]
                if mode == "peer":
                    ops.pass_a(x, r, p_in, p_out, ap, scratch)
                elif mode == "off":
                    halo(r) if k == 0 else halo(r, p_in)
                    ops.pass_a(x, r, p_in, p_out, ap, scratch)
                elif mode == "pipeline":
                    halo.wait(halo.start(r) + pending_p)
                    ops.pass_a(x, r, p_in, p_out, ap, scratch)
                else:  # split
                    works = halo.start(r)
                    ops.pass_a_range(x, r, p_in, p_out, ap, scratch, g, nz - 2 * g, False)
                    halo.wait(works + pending_p)
                    ops.pass_a_range(x, r, p_in, p_out, ap, scratch, 0, g, True)
                    ops.pass_a_range(x, r, p_in, p_out, ap, scratch, nz - g, g, True)
                pending_p = halo.start(p_out) if mode not in ("off", "peer") else []
                ops.reduce(scratch, 1, 1)
                ops.pass_b(r, ap, scratch)
                ops.reduce(scratch, 2, 2)
                k += 1
            rep, active = ops.read(scratch)
    finally:
        halo.wait(pending_p)
        if hasattr(ops, "use_peers"):
            ops.use_peers(False)
    ops.flush_x(x, pring, scratch)  # the last iteration's x update
    return rep, time.perf_counter() - t0


class DistributedOperator:
    """This rank's slab of a b200 operator (constant-coefficient box system).

    ``pcg_device`` / ``apply_device`` take ghosted-slab tensors of this rank;
    ``scatter`` / ``gather`` move reference-shaped host arrays in and out.
    """

    strategy = "b200-zslab"

    def __init__(self, data, group=None, device=None):
        import torch
        import torch.distributed as dist

        from .device import NativePlan, SlabLayout, require_cuda

        self.data = data
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = require_cuda(device)
        nzg, ny, nx = data.dims3
        self.part = SlabPartition(nzg, self.world, self.rank)
        self.part.check_min(data.n_b)
        self.layout = SlabLayout(self.part.nz, ny, nx, ghost=data.n_b,
                                 z_offset=self.part.z_offset, nz_global=nzg)
        self._plans = {}
        torch.cuda.set_device(self.device)
        # halos get their own communicator (own NCCL stream), so p_k's
        # exchange overlaps the scalar all-reduce and pass B ("pipeline")
        self.halo_group = group
        if self.world > 1:
            ranks = dist.get_process_group_ranks(group) if group is not None else None
            self.halo_group = dist.new_group(ranks=ranks)
        self.halo = HaloExchanger(self.layout, self.rank, self.world, self.halo_group)
        self._work = None

    def plan(self, precond="jacobi"):
        from .device import NativePlan

        if precond not in self._plans:
            self._plans[precond] = NativePlan(self.data, self.layout, self.device, precond)
        return self._plans[precond]

    # -- data movement ---------------------------------------------------
    def scatter(self, full):
        """Reference-shaped host array -> this rank's ghosted slab (device)."""
        full = np.asarray(full, dtype=np.float64).reshape(self.data.dims3)
        lo, hi = self.part.bounds()
        return self.layout.upload(full[lo:hi], self.device)

    def gather(self, buf):
        """All ranks' owned planes -> full array on every rank (host)."""
        import torch
        import torch.distributed as dist

        own = self.layout.owned(buf).contiguous()
        if self.world == 1:
            return own.cpu().numpy().reshape(self.data.cext)
        sizes = [self.part.bounds(r) for r in range(self.world)]
        maxz = max(hi - lo for lo, hi in sizes)
        pad = torch.zeros((maxz,) + tuple(own.shape[1:]), dtype=own.dtype, device=own.device)
        pad[: own.shape[0]] = own
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        out = torch.cat([parts[r][: hi - lo] for r, (lo, hi) in enumerate(sizes)])
        return out.cpu().numpy().reshape(self.data.cext)

    # -- operator / solver ------------------------------------------------
    def apply_device(self, c_buf, out_buf):
        self.halo(c_buf)
        self.plan().apply(c_buf, out_buf)
        return out_buf

    def mass_apply_device(self, c_buf, out_buf, f_buf=None, a=0.0, cm=None):
        self.halo(c_buf)
        cm = self.data.vol if cm is None else cm
        self.plan().mass_apply(c_buf, f_buf, cm, a, out_buf)
        return out_buf

    def _work_buffers(self, max_iter):
        import torch

        if self._work is None:
            from .device import choose_ring

            lay = self.layout
            ring = choose_ring(lay, self.device)
            self._work = dict(r=lay.alloc(self.device), pring=lay.alloc_ring(self.device, ring),
                              ap=lay.alloc(self.device), scratch=self.plan().scratch(),
                              history=None)
            self._peers = self._map_peers(self._work)
        w = self._work
        if w["history"] is None or w["history"].numel() < max_iter + 1:
            w["history"] = torch.zeros(max_iter + 1, dtype=torch.float64, device=self.device)
        return w

    def _map_peers(self, w):
        """Map the neighbours' p ring and r (CUDA IPC: NVLink peer memory
        across GPUs, the same device in the one-GPU multi-process test) for
        the "peer" halo mode.  Every rank must succeed or none uses it."""
        import torch.distributed as dist

        from . import _native as N
        from .device import ipc_close, ipc_export, ipc_import

        if self.world == 1 or os.environ.get("BSPDE_PEER_HALO", "1") == "0":
            return None
        ring, r = w["pring"], w["r"]
        try:
            mine = dict(ring=ipc_export(ring), r=ipc_export(r), stride=int(ring.stride(0)),
                        nz=self.layout.nz)
        except Exception:  # noqa: BLE001 - no IPC on this platform: NCCL halos
            mine = None
        info = [None] * self.world
        dist.all_gather_object(info, mine, group=self.group)
        opened, ok = [], all(v is not None for v in info)
        nb = {}
        if ok:
            try:
                for side, q in (("lo", self.rank - 1), ("hi", self.rank + 1)):
                    if 0 <= q < self.world:
                        pr = ipc_import(*info[q]["ring"])
                        opened.append(pr)
                        rr = ipc_import(*info[q]["r"])
                        opened.append(rr)
                        nb[side] = (pr, info[q]["stride"], rr, info[q]["nz"])
            except Exception:  # noqa: BLE001
                ok = False
        flags = [None] * self.world
        dist.all_gather_object(flags, ok, group=self.group)
        if not all(flags):
            for ptr in opened:
                ipc_close(ptr)
            return None
        self._peer_maps = opened
        lo, hi = nb.get("lo"), nb.get("hi")
        return N.SlabPeers(ring=ring.data_ptr(), r=r.data_ptr(), ring_stride=int(ring.stride(0)),
                           ring_len=int(ring.shape[0]), lo_nz=lo[3] if lo else 0,
                           lo_ring=lo[0] if lo else None, lo_ring_stride=lo[1] if lo else 0,
                           lo_r=lo[2] if lo else None, hi_ring=hi[0] if hi else None,
                           hi_ring_stride=hi[1] if hi else 0, hi_r=hi[2] if hi else None)

    def rhs_buffer(self, max_iter=1000):
        """The heat RHS b shares the CG's Ap field (b is dead once r0 = b - A x0
        is formed), as in the single-GPU HeatSolver."""
        return self._work_buffers(max_iter)["ap"]

    def pcg_device(self, b_buf, x_buf, config: SolveConfig = None, has_x0=True):
        config = config or SolveConfig()
        w = self._work_buffers(config.max_iter)
        ops = NativeSlabOps(self.plan(config.precond), self.world, self.group,
                            peers=getattr(self, "_peers", None))
        rep, wall = distributed_pcg(ops, self.halo, b_buf, x_buf, w["r"],
                                    w["pring"], w["ap"], w["scratch"], config, has_x0,
                                    w["history"] if config.record_history else None)
        return report_from(rep, config, wall, w["history"])

    def heat_step_device(self, u_buf, F_buf, dt, config: SolveConfig = None):
        """One implicit-Euler step in place on this rank's slab, x0 = u: the
        right-hand side vol M u + dt F is fused into the first residual
        (``bspde_heat_residual``), as in the single-GPU ``bspde_heat_step``."""
        config = config or SolveConfig()
        w = self._work_buffers(config.max_iter)
        ops = NativeSlabOps(self.plan(config.precond), self.world, self.group,
                            peers=getattr(self, "_peers", None))
        rep, wall = distributed_pcg(ops, self.halo, None, u_buf, w["r"], w["pring"], w["ap"],
                                    w["scratch"], config, True,
                                    w["history"] if config.record_history else None,
                                    heat=(F_buf, self.data.vol, dt))
        return report_from(rep, config, wall, w["history"])

    def pcg_host(self, rhs, config, x0=None):
        b = self.scatter(rhs)
        x = self.scatter(x0) if x0 is not None else self.layout.alloc(self.device)
        rep = self.pcg_device(b, x, config, has_x0=x0 is not None)
        return self.gather(x), rep
