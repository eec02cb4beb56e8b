"""Multi-rank z-slab CG orchestration on CPU (gloo, world_size 2 and 3).

The product's distributed driver (``distributed.distributed_pcg``, the slab
partition and the halo exchanger) runs unchanged; only the per-slab kernels
are replaced by a CPU test double with the same semantics as the sm_100a
step-wise entry points (pass A / pass B / finalize, fuse = 0), built on the
oracle operator.  The gathered solution must match the single-process oracle
pcg.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bspde_oracle as O
from paper_1904_03057_b200.device import SlabLayout
from paper_1904_03057_b200.distributed import HaloExchanger, SlabPartition, distributed_pcg
from paper_1904_03057_b200.solver import SolveConfig


class CpuSlabOps:
    """CPU stand-in for NativeSlabOps: same vectors, same scalar state machine."""

    def __init__(self, ora, layout, precond="jacobi"):
        self.ora, self.lay = ora, layout
        diag = ora.jacobi_diagonal()
        inv = np.where(diag != 0, 1.0 / diag, 1.0) if precond == "jacobi" else np.ones_like(diag)
        g = layout.ghost
        full_inv = np.zeros((ora.cext[0] + 2 * g,) + ora.cext[1:])
        full_inv[g:g + ora.cext[0]] = inv
        lo = layout.z_offset
        self.inv = torch.from_numpy(full_inv[lo:lo + layout.nz + 2 * g].copy())
        self.state = {}

    def _own(self, t):
        return self.lay.owned(t)

    def _apply(self, c):
        """A c for the owned planes, using ghost planes (embed in a global array)."""
        g, lo, nz = self.lay.ghost, self.lay.z_offset, self.lay.nz
        nzg = self.ora.cext[0]
        full = np.zeros((nzg + 2 * g,) + self.ora.cext[1:])
        full[lo:lo + nz + 2 * g] = c[:, :, : self.lay.nx].numpy()
        out = self.ora.apply(full[g:g + nzg])
        return torch.from_numpy(out[lo:lo + nz].copy())

    def reduce(self, scratch, n, kind):
        """NativeSlabOps.reduce: combine the ranks' sums, then the scalar update
        (a plain all-reduce here; the product all-gathers double-double pairs)."""
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(scratch[:n])
        self.finalize(scratch, kind)

    def setup(self, scratch, history, cfg, has_x0, ring=4):
        self.state = dict(tol=cfg.tol, max_iter=cfg.max_iter, has_x0=has_x0, it=0, active=1,
                          alpha_ring=[0.0] * ring)

    def residual(self, b, x, r, scratch):
        ax = self._apply(x)
        rv = self._own(b) - ax
        self._own(r).copy_(rv)
        own_inv = self.inv[self.lay.ghost:self.lay.ghost + self.lay.nz, :, : self.lay.nx]
        scratch[0] = float((self._own(b) ** 2).sum())
        scratch[1] = float((rv * (own_inv * rv)).sum())
        scratch[2] = float((rv ** 2).sum())

    def _x_update(self, x, p_in):
        """x += alpha_{k-1} p_{k-1} (pass A of iteration k >= 1, as the kernel)."""
        s = self.state
        if s["it"] >= 1 and not s.get("x_applied_in", -1) == s["it"]:
            self._own(x).add_(s["alpha"] * self._own(p_in))
            s["x_applied_in"] = s["it"]

    def pass_a(self, x, r, p_in, p_out, ap, scratch):
        s = self.state
        if not s["active"]:
            return
        self._x_update(x, p_in)
        g, nz, nx = self.lay.ghost, self.lay.nz, self.lay.nx
        pn = r[:, :, :nx] * self.inv + s["beta"] * p_in[:, :, :nx]
        self._own(p_out).copy_(pn[g:g + nz])
        apv = self._apply(torch.nn.functional.pad(pn, (0, p_in.shape[2] - nx)))
        self._own(ap).copy_(apv)
        scratch[0] = float((pn[g:g + nz] * apv).sum())

    def pass_a_range(self, x, r, p_in, p_out, ap, scratch, z0, cnt, accumulate):
        """bspde_cg_pass_a_range: only owned planes [z0, z0 + cnt) are
        produced; the interior range is called while the ghosts are still in
        flight, so outputs there must not depend on them (banded in z)."""
        s = self.state
        if not s["active"]:
            return
        g, nz, nx = self.lay.ghost, self.lay.nz, self.lay.nx
        self.range_calls = getattr(self, "range_calls", 0) + 1
        self._x_update(x, p_in)  # (the kernel updates each range's planes; same result)
        pn = r[:, :, :nx] * self.inv + s["beta"] * p_in[:, :, :nx]
        apv = self._apply(torch.nn.functional.pad(pn, (0, p_in.shape[2] - nx)))
        sl = slice(z0, z0 + cnt)
        self._own(p_out)[sl] = pn[g:g + nz][sl]
        self._own(ap)[sl] = apv[sl]
        part = float((pn[g:g + nz][sl] * apv[sl]).sum())
        scratch[0] = (float(scratch[0]) if accumulate else 0.0) + part

    def pass_b(self, r, ap, scratch):
        s = self.state
        if not s["active"]:
            return
        g, nz, nx = self.lay.ghost, self.lay.nz, self.lay.nx
        own_inv = self.inv[g:g + nz, :, :nx]
        self._own(r).sub_(s["alpha"] * self._own(ap))
        rv = self._own(r)
        scratch[0] = float((rv * (own_inv * rv)).sum())
        scratch[1] = float((rv ** 2).sum())

    def finalize(self, scratch, kind):
        s = self.state
        if kind == 0:
            bb, rz, rr = (float(v) for v in scratch[:3])
            s["scale"] = np.sqrt(bb) if bb > 0 else 1.0
            s["rz"], s["res"], s["beta"] = rz, np.sqrt(rr), 0.0
            s["res0"] = s["res"]
            if bb == 0 and not s["has_x0"]:
                s["active"] = 0
                return
        elif not s["active"]:
            return
        elif kind == 1:
            s["x_done"] = s["it"]
            pAp = float(scratch[0])
            if pAp <= 0:
                s["active"] = 0
                return
            s["alpha"] = s["rz"] / pAp
            return
        else:
            rz_new, rr = float(scratch[0]), float(scratch[1])
            ring = s.setdefault("alpha_ring", [0.0] * 4)
            ring[s["it"] % len(ring)] = s["alpha"]
            s["beta"] = rz_new / s["rz"]
            s["rz"] = rz_new
            s["res"] = np.sqrt(rr)
            s["it"] += 1
        s["active"] = int(s["res"] / s["scale"] > s["tol"] and s["it"] < s["max_iter"])

    def flush_x(self, x, pring, scratch):
        s = self.state
        R = pring.shape[0]
        ring = s.get("alpha_ring", [0.0] * R)
        for j in range(s.get("x_done", 0), s["it"]):  # the last iteration's update
            self._own(x).add_(ring[j % R] * self._own(pring[j % R]))
        s["x_done"] = s["it"]

    def read(self, scratch):
        class Rep:
            pass

        rep = Rep()
        rep.iterations = self.state["it"]
        rep.relative_residual = self.state["res"] / self.state["scale"]
        return rep, bool(self.state["active"])


def _worker(rank, world, port, ext, p, out_q, overlap="pipeline", ring=4):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BSPDE_HALO_OVERLAP=overlap)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        step = tuple(1.0 / (n - 1) for n in ext)
        ora = O.KronOperator(ext, step, p, 0.02, 1.0)
        part = SlabPartition(ora.cext[0], world, rank)
        part.check_min(p)
        lay = SlabLayout(part.nz, ora.cext[1], ora.cext[2], ghost=p, z_offset=part.z_offset,
                         nz_global=ora.cext[0])
        rng = np.random.default_rng(0)
        axes = [np.linspace(0, 1, n) for n in ora.cext]
        Z, Y, X = np.meshgrid(*axes, indexing="ij")
        b_full = ora.mass_apply(np.cos(3 * Z) * np.sin(2 * Y + 0.3) + np.exp(-5 * (X - 0.4) ** 2))
        x0_full = 0.1 * rng.normal(size=ora.cext)
        lo, hi = part.bounds()
        b = lay.upload(b_full[lo:hi], "cpu")
        x = lay.upload(x0_full[lo:hi], "cpu")
        r, ap = lay.alloc("cpu"), lay.alloc("cpu")
        pring = torch.zeros((ring,) + tuple(lay.buf_shape), dtype=torch.float64)
        scratch = torch.zeros(8, dtype=torch.float64)
        ops = CpuSlabOps(ora, lay)
        halo = HaloExchanger(lay, rank, world, dist.new_group())  # own communicator, as the product

        cfg = SolveConfig(tol=1e-13, max_iter=1000, poll_every=3)
        rep, _ = distributed_pcg(ops, halo, b, x, r, pring, ap, scratch, cfg, has_x0=True)
        own = lay.owned(x).contiguous()
        parts = [torch.zeros((part.bounds(q)[1] - part.bounds(q)[0],) + tuple(own.shape[1:]),
                             dtype=own.dtype) for q in range(world)]
        parts[rank].copy_(own)
        for q in range(world):
            dist.broadcast(parts[q], src=q)
        if rank == 0:
            xs = torch.cat(parts).numpy()
            xo, ro = O.pcg(ora.apply, ora.jacobi_diagonal, b_full, tol=1e-13, max_iter=1000,
                           x0=x0_full)
            out_q.put((rep.iterations, ro["iterations"],
                       float(np.linalg.norm(xs - xo) / np.linalg.norm(xo)),
                       getattr(ops, "range_calls", 0), lay.nz))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,ext,overlap,ring", [
    (2, (13, 10, 11), "split", 4),     # 15 coefficient planes: slabs of 8 / 7, both split pass A
    (3, (17, 9, 10), "split", 4),      # 19: 7 / 6 / 6, only rank 0 has an interior range (> 2p)
    (3, (13, 9, 10), "split", 4),      # 15: 5 / 5 / 5, no interior range: pipeline instead
    (2, (13, 10, 11), "pipeline", 4),  # p_k's exchange in flight under the all-reduce + pass B
    (3, (17, 9, 10), "pipeline", 4),
    (2, (21, 9, 10), "off", 4),        # both exchanges before pass A
    (2, (13, 10, 11), "pipeline", 2),  # two-field search-direction ring (x every 2nd pass B)
])
def test_zslab_cg_matches_single_process(world, ext, overlap, ring):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ext, 3, q, overlap, ring))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    its, its_o, rel, range_calls, nz0 = q.get(timeout=10)
    assert abs(its - its_o) <= 1, (its, its_o)
    assert rel < 1e-10, rel
    split = overlap == "split" and nz0 > 2 * 3  # rank 0's slab has an interior range
    assert (range_calls > 0) == split, range_calls


def test_partition_bounds():
    part = SlabPartition(930, 8, 0)
    spans = [part.bounds(r) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 930
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(Exception):
        SlabPartition(5, 8, 0)
    with pytest.raises(Exception):
        SlabPartition(10, 4, 0).check_min(3)


def test_halo_mode_selection(monkeypatch):
    """BSPDE_HALO_OVERLAP: single rank -> off; pipeline default; split needs a
    ranged pass A and an interior range (> 2p planes), else pipeline; bad
    values raise ConfigurationError."""
    from paper_1904_03057_b200.distributed import _halo_mode
    from paper_1904_03057_b200.errors import ConfigurationError

    class Ops:
        def pass_a_range(self, *a):
            pass

    def halo(nz, world=2):
        return HaloExchanger(SlabLayout(nz, 5, 6, ghost=3, z_offset=0, nz_global=2 * nz),
                             0, world)

    monkeypatch.delenv("BSPDE_HALO_OVERLAP", raising=False)
    assert _halo_mode(Ops(), halo(10, world=1)) == "off"
    assert _halo_mode(Ops(), halo(10)) == "pipeline"
    monkeypatch.setenv("BSPDE_HALO_OVERLAP", "split")
    assert _halo_mode(Ops(), halo(10)) == "split"
    assert _halo_mode(Ops(), halo(6)) == "pipeline"      # no interior range
    assert _halo_mode(object(), halo(10)) == "pipeline"  # no ranged pass A
    monkeypatch.setenv("BSPDE_HALO_OVERLAP", "0")
    assert _halo_mode(Ops(), halo(10)) == "off"
    monkeypatch.setenv("BSPDE_HALO_OVERLAP", "sideways")
    with pytest.raises(ConfigurationError):
        _halo_mode(Ops(), halo(10))
