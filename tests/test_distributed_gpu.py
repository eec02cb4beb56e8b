"""The native z-slab solver with several processes on the one GPU.

2 and 3 ranks on cuda:0 run ``DistributedOperator.pcg_device`` --
``NativeSlabOps`` (the sm_100a step-wise kernels with fuse = 0: ranged pass
A, pass B, the 1-thread finalize) driven by ``distributed_pcg`` -- over the
gloo backend, whose halo planes and scalar all-gathers are staged through
host memory (NCCL refuses two ranks on one device), and the "peer" mode
in which pass B stores the halo planes of r and p_k into the neighbours'
fields mapped by CUDA IPC (the same device here; NVLink peer memory across GPUs).
Every halo mode and both ring lengths; the gathered solution must equal the fused
single-rank solver's bit for bit (same iteration count) and match the oracle
(counts +-1, coefficients 1e-10 at tol 1e-13).  The ranks' kernels never wait on one another (the exchanges are
synchronous host copies), so sharing the device is safe.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _system(ext, p):
    from paper_1904_03057_b200 import BoxDomain, Grid, build_system

    step = tuple(1.0 / (n - 1) for n in ext)
    return build_system(BoxDomain(Grid(ext, step)), p, p, 0.02, 1.0, []), step


def _inputs(ext, p):
    """b = M g for a smooth g (an assembled right-hand side: a raw smooth
    array is far outside the range of the degree-5 mass matrix, and the
    reference recurrence's divergence guard fires at iteration 1 on it),
    x0 a smooth field."""
    from oracle import bspde_oracle as O

    step = tuple(1.0 / (n - 1) for n in ext)
    ora = O.KronOperator(ext, step, p, 0.02, 1.0)
    axes = [np.linspace(0, 1, n) for n in ora.cext]
    Z, Y, X = np.meshgrid(*axes, indexing="ij")
    b = ora.mass_apply(np.cos(3 * Z) * np.sin(2 * Y + 0.3) + np.exp(-5 * (X - 0.4) ** 2))
    x0 = 0.1 * np.sin(2 * Z + 1) * np.cos(3 * X) * Y  # smooth: p = 5 stagnates on noise
    return b, x0


def _worker(rank, world, port, ext, p, mode, ring, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BSPDE_HALO_OVERLAP=mode,
                      BSPDE_P_RING_LEN=str(ring))
    import torch
    import torch.distributed as dist

    from paper_1904_03057_b200 import SolveConfig
    from paper_1904_03057_b200.distributed import DistributedOperator

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data, _ = _system(ext, p)
        op = DistributedOperator(data, device=0)
        b_full, x0_full = _inputs(ext, p)
        b = op.scatter(b_full)
        its = []
        for tol in (1e-10, 1e-13):  # counts at the north_star tol; coefficients at 1e-13
            x = op.scatter(x0_full)
            rep = op.pcg_device(b, x, SolveConfig(tol=tol, max_iter=2000, poll_every=3),
                                has_x0=True)
            its.append(rep.iterations)
        xs = op.gather(x)
        # a distributed apply through the same halo path
        t = op.gather(op.apply_device(op.scatter(x0_full), op.layout.alloc(op.device)))
        # one heat step (RHS fused into the first residual), u0 = x0, F = b
        u = op.scatter(x0_full)
        hrep = op.heat_step_device(u, op.scatter(b_full), 0.01,
                                   SolveConfig(tol=1e-12, max_iter=2000, poll_every=3))
        hs = op.gather(u)
        peer = op._peers is not None
        if rank == 0:
            q.put((its, xs, t, int(op._work["pring"].shape[0]), op.layout.nz, peer,
                   hrep.iterations, hs))
    finally:
        dist.destroy_process_group()


CASES = [
    (2, (24, 20, 22), 3, "peer", 2),      # halos stored by pass B through IPC
    (3, (24, 20, 22), 3, "peer", 4),
    (3, (16, 18, 17), 1, "peer", 2),      # p = 1: one ghost plane per side
    (2, (24, 20, 22), 3, "pipeline", 4),
    (3, (24, 20, 22), 3, "split", 4),     # 26 planes: slabs 9 / 9 / 8, interior ranges
    (2, (24, 20, 22), 3, "off", 2),       # two-field ring
    (3, (16, 18, 17), 1, "pipeline", 2),  # p = 1: one ghost plane
    (2, (20, 17, 19), 2, "split", 4),     # p = 2: even degree, ghost = 2
]
# (p >= 4 stagnate near 1e-11 / 1e-9 with Jacobi here; their ranged pass A is
# checked bitwise on emulated slabs in test_parity_gpu.py)


@pytest.mark.parametrize("world,ext,p,mode,ring", CASES)
def test_native_zslab_multiprocess(cuda_device, world, ext, p, mode, ring):
    import torch.multiprocessing as mp

    from oracle import bspde_oracle as O
    from paper_1904_03057_b200 import SolveConfig, make_operator, pcg

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ext, p, mode, ring, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    its, xs, t, ring_used, nz0, peer, h_its, hs = res
    assert ring_used == ring
    assert peer  # the neighbours' fields were mapped (CUDA IPC on the one device)
    data, step = _system(ext, p)
    b_full, x0_full = _inputs(ext, p)
    # fused single-rank solver and the oracle recurrence on the same inputs:
    # counts +-1 at tol 1e-10; at tol 1e-13 (hundreds of iterations) +-max(1, 1%)
    # and the coefficients to 1e-10
    op = make_operator(data, "b200")
    ora = O.KronOperator(ext, step, p, 0.02, 1.0)
    for k, tol in enumerate((1e-10, 1e-13)):
        x1, rep1 = pcg(op, b_full, SolveConfig(tol=tol, max_iter=2000), x0=x0_full)
        xo, ro = O.pcg(ora.apply, ora.jacobi_diagonal, b_full, tol=tol, max_iter=2000,
                       x0=x0_full)
        bar = 1 if k == 0 else max(1, round(0.01 * ro["iterations"]))
        assert abs(its[k] - rep1.iterations) <= bar, (tol, its[k], rep1.iterations)
        assert abs(its[k] - ro["iterations"]) <= bar, (tol, its[k], ro["iterations"])
    # the ranks' double-double pairs are combined before rounding, so the slab
    # solve reproduces the single-device iterates bit for bit
    assert its[1] == rep1.iterations
    assert np.array_equal(xs, x1), np.abs(xs - x1).max()
    assert np.linalg.norm(xs - x1) / np.linalg.norm(x1) < 1e-10
    assert np.linalg.norm(xs - xo) / np.linalg.norm(xo) < 1e-10
    want = ora.apply(x0_full)
    assert np.abs(t - want).max() / np.abs(want).max() < 1e-13
    # the distributed heat step equals the single-GPU bspde_heat_step bit for bit
    import torch

    from paper_1904_03057_b200.heat import heat_step_device

    lay = op.layout
    u1 = lay.upload(x0_full, op.device)
    F1 = lay.upload(b_full, op.device)
    rep1 = heat_step_device(op, u1, F1, 0.01, SolveConfig(tol=1e-12, max_iter=2000))
    assert h_its == rep1.iterations
    assert np.array_equal(hs, lay.download(u1))
    del u1, F1
    torch.cuda.empty_cache()
