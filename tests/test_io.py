"""TBSF tensor files: reader/writer against files the reference wrote
(tests/golden/tbsf, make_golden.py ``tbsf``) and the reference's own
``test_io.py:40-75`` checks; device checkpoints on the GPU."""

import os
import struct

import numpy as np
import pytest

from paper_1904_03057_b200.errors import FormatError
from paper_1904_03057_b200.io import read_tensor, write_tensor

GOLD = os.path.join(os.path.dirname(__file__), "golden", "tbsf")
CASES = (("f8_3d_p3", (5, 7, 3), np.float64, 3),
         ("f4_2d", (3, 4), np.float32, -1),
         ("f8_1d_p5", (11,), np.float64, 5))


def _expected(shape, dtype):
    n = int(np.prod(shape))
    return (np.arange(n, dtype=np.float64) * 0.37 - 1.5).reshape(shape).astype(dtype)


@pytest.mark.parametrize("name,shape,dtype,deg", CASES)
def test_reads_reference_files(name, shape, dtype, deg):
    arr, d = read_tensor(os.path.join(GOLD, name + ".tbsf"))
    assert d == deg and arr.dtype == np.dtype(dtype) and arr.shape == shape
    assert np.array_equal(arr, _expected(shape, dtype))


@pytest.mark.parametrize("name,shape,dtype,deg", CASES)
def test_writes_reference_bytes(tmp_path, name, shape, dtype, deg):
    p = tmp_path / "t.tbsf"
    write_tensor(p, _expected(shape, dtype), degree=deg)
    with open(os.path.join(GOLD, name + ".tbsf"), "rb") as f:
        assert p.read_bytes() == f.read()


def test_roundtrip_f64_bit_exact(tmp_path):
    arr = np.random.default_rng(0).normal(size=(5, 7, 3))
    p = tmp_path / "t.tbsf"
    write_tensor(p, arr, degree=3)
    back, deg = read_tensor(p)
    assert deg == 3 and back.dtype == np.float64 and np.array_equal(back, arr)


def test_roundtrip_f32_and_torch_input(tmp_path):
    import torch

    arr = np.arange(12, dtype=np.float32).reshape(3, 4)
    p = tmp_path / "t.tbsf"
    write_tensor(p, torch.from_numpy(arr))
    back, deg = read_tensor(p)
    assert deg == -1 and back.dtype == np.float32 and np.array_equal(back, arr)
    write_tensor(p, np.arange(6, dtype=np.int32))  # non-f4 dtypes are stored as f8
    back, _ = read_tensor(p)
    assert back.dtype == np.float64 and np.array_equal(back, np.arange(6))


def test_truncated_payload_names_lengths(tmp_path):
    p = tmp_path / "t.tbsf"
    write_tensor(p, np.ones((4, 4)))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(FormatError) as exc:
        read_tensor(p)
    assert "120" in str(exc.value) and "128" in str(exc.value)
    assert exc.value.offset == 12 + 16 + 2


@pytest.mark.parametrize("blob,offset", [
    (b"NOPE" + b"\0" * 32, 0),
    (struct.pack("<4sII", b"TBSF", 2, 1) + b"\0" * 16, 4),
    (struct.pack("<4sII", b"TBSF", 1, 4) + b"\0" * 40, 8),
    (struct.pack("<4sII", b"TBSF", 1, 0), 8),
    (b"TBSF\1\0", 6),
    (struct.pack("<4sII", b"TBSF", 1, 2) + b"\0" * 8, 20),
    (struct.pack("<4sIIQBb", b"TBSF", 1, 1, 1, 7, 0) + b"\0" * 8, 20),
])
def test_header_errors_carry_offsets(tmp_path, blob, offset):
    p = tmp_path / "bad.tbsf"
    p.write_bytes(blob)
    with pytest.raises(FormatError) as exc:
        read_tensor(p)
    assert exc.value.offset == offset


def test_failed_write_leaves_no_file(tmp_path):
    class Boom:
        def __array__(self, dtype=None, copy=None):
            raise RuntimeError("boom")

    p = tmp_path / "t.tbsf"
    with pytest.raises(RuntimeError):
        write_tensor(p, Boom())
    assert list(tmp_path.iterdir()) == []


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_field_checkpoint_roundtrip(tmp_path):
    import torch

    from paper_1904_03057_b200.device import SlabLayout
    from paper_1904_03057_b200.io import read_field, write_field

    lay = SlabLayout(nz=9, ny=6, nx=5, ghost=3)
    dev = torch.device("cuda", 0)
    host = np.random.default_rng(1).normal(size=lay.owned_shape)
    buf = lay.upload(host, dev)
    p = tmp_path / "f.tbsf"
    write_field(p, lay, buf, degree=3)
    arr, deg = read_tensor(p)
    assert deg == 3 and np.array_equal(arr, host)
    back, deg = read_field(p, lay, dev, degree=3)
    assert torch.equal(back, buf)  # ghosts and pitch padding stay zero
    with pytest.raises(FormatError):
        read_field(p, lay, dev, degree=2)
    with pytest.raises(FormatError):
        read_field(p, SlabLayout(nz=8, ny=6, nx=5, ghost=3), dev)
    write_tensor(p, host.astype(np.float32), degree=3)  # f4 files load widened
    back, _ = read_field(p, lay, dev)
    assert np.array_equal(lay.download(back), host.astype(np.float32).astype(np.float64))


@pytest.mark.gpu
def test_heat_solver_save_restore_continues_bitwise(tmp_path):
    from paper_1904_03057_b200 import Grid, HeatProblem, HeatSolver
    from paper_1904_03057_b200.solver import SolveConfig

    n = 12
    h = 1.0 / (n - 1)
    cfg = SolveConfig(tol=1e-12, max_iter=500)

    def problem():
        return HeatProblem(grid=Grid((n,) * 3, (h,) * 3), degree=3, dt=4 * h * h,
                           initial=lambda x, y, z: np.sin(np.pi * x) * np.cos(y) + z,
                           source=1.0)

    ref = HeatSolver(problem(), cfg)
    ref.run(4)
    s1 = HeatSolver(problem(), cfg)
    s1.run(2)
    p = tmp_path / "ck.tbsf"
    s1.save(p)
    s2 = HeatSolver(problem(), cfg)
    s2.restore(p)
    s2.run(2)
    assert np.array_equal(s2.coefficients(), ref.coefficients())


# ---------------------------------------------------------------- mask / VTK
def test_mask_file_roundtrip_and_reference_bytes(tmp_path):
    from paper_1904_03057_b200.io import read_mask, write_mask

    vol = (np.arange(4 * 5 * 6) * 7 % 256).astype(np.uint8).reshape(4, 5, 6)
    occ, thr = read_mask(os.path.join(GOLD, "vol_4x5x6.tbsm"))
    assert thr == 100 and np.array_equal(occ, vol >= 100)
    p = tmp_path / "m.tbsm"
    write_mask(p, vol, threshold=100)
    with open(os.path.join(GOLD, "vol_4x5x6.tbsm"), "rb") as f:
        assert p.read_bytes() == f.read()


def test_mask_file_errors(tmp_path):
    from paper_1904_03057_b200.io import read_mask, write_mask

    p = tmp_path / "m.tbsm"
    write_mask(p, np.ones((3, 3), dtype=np.uint8))
    p.write_bytes(p.read_bytes() + b"\1")
    with pytest.raises(FormatError):
        read_mask(p)
    p.write_bytes(b"TBSM v1\nextents 2 2\n")
    with pytest.raises(FormatError) as exc:
        read_mask(p)
    assert exc.value.offset == 0
    p.write_bytes(b"NOPE v1\nextents 1\nthreshold 1\n\1")
    with pytest.raises(FormatError):
        read_mask(p)


def test_vtk_export_matches_reference_text(tmp_path):
    from paper_1904_03057_b200.domain import Grid
    from paper_1904_03057_b200.errors import ValidationError
    from paper_1904_03057_b200.io import export_vtk

    f3 = (np.arange(24, dtype=np.float64).reshape(3, 4, 2) - 7.5) / 3.0
    export_vtk(tmp_path / "a.vtk", f3, Grid((3, 4, 2), (0.5, 1.0, 2.0), (1.0, -2.0, 0.25)),
               name="temp")
    f2 = np.cos(np.arange(12, dtype=np.float64)).reshape(3, 4)
    export_vtk(tmp_path / "b.vtk", f2, Grid((3, 4), (0.5, 1.0)))
    for mine, ref in (("a.vtk", "field3.vtk"), ("b.vtk", "field2.vtk")):
        with open(os.path.join(GOLD, ref)) as f:
            assert (tmp_path / mine).read_text() == f.read()
    with pytest.raises(ValidationError):
        export_vtk(tmp_path / "c.vtk", np.zeros(4), Grid((4,), (1.0,)))


@pytest.mark.gpu
def test_heat_solver_2d_checkpoint_uses_problem_extents(tmp_path):
    """A 2-D heat problem saves its real (ny, nx) coefficient extents (not the
    padded (1, ny, nx) device layout) and restores a file the reference's
    write_tensor wrote for that array."""
    from paper_1904_03057_b200 import Grid, HeatProblem, HeatSolver
    from paper_1904_03057_b200.solver import SolveConfig

    n = 14
    h = 1.0 / (n - 1)
    hs = HeatSolver(HeatProblem(grid=Grid((n, n), (h, h)), degree=3, dt=4 * h * h,
                                initial=lambda x, y: np.sin(np.pi * x) * np.cos(y)),
                    SolveConfig(tol=1e-12, max_iter=500))
    hs.run(1)
    p = tmp_path / "c2.tbsf"
    hs.save(p)
    arr, deg = read_tensor(p)
    assert arr.shape == hs.data.cext and deg == 3
    assert np.array_equal(arr, hs.coefficients())
    q = tmp_path / "ref.tbsf"
    want = np.random.default_rng(3).normal(size=hs.data.cext)
    write_tensor(q, want, degree=3)  # the reference's writer (byte-identical, tests above)
    hs.restore(q)
    assert np.array_equal(hs.coefficients(), want)
