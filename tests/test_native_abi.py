"""The C ABI library loads (no GPU needed) and matches include/bspde_b200.h."""

import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1904_03057_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bspde_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bspde_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_symbol():
    lib = N.load()
    decl = declared_functions()
    assert len(decl) >= 15
    bound = {name for name, _, _ in N.SIGNATURES}
    missing_binding = set(decl) - bound
    assert not missing_binding, f"header functions without ctypes binding: {missing_binding}"
    for name in decl:
        assert hasattr(lib, name), f"{name} not exported by {N.LIB_PATH}"
    assert lib.bspde_version() >= 1


def test_error_path_without_gpu():
    lib = N.load()
    h = C.c_void_p()
    rc = lib.bspde_plan_create(None, C.byref(h))
    assert rc != 0
    assert b"null" in lib.bspde_last_error()


@pytest.mark.skipif(not os.path.exists("/usr/bin/gcc"), reason="gcc missing")
def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
#define F(T, f) printf("%s.%s %zu\\n", #T, #f, offsetof(T, f));
int main(void) {{
  printf("bspde_plan_desc %zu\\n", sizeof(bspde_plan_desc));
  printf("bspde_cg_config %zu\\n", sizeof(bspde_cg_config));
  printf("bspde_cg_report %zu\\n", sizeof(bspde_cg_report));
  F(bspde_plan_desc, pitch_y) F(bspde_plan_desc, mass_table) F(bspde_plan_desc, inv_diag_table)
  F(bspde_plan_desc, c_mass) F(bspde_plan_desc, c_stiff) F(bspde_plan_desc, ew)
  F(bspde_cg_config, poll_every) F(bspde_cg_report, relative_residual)
  F(bspde_cg_report, last_pAp)
  printf("bspde_stencil_desc %zu\\n", sizeof(bspde_stencil_desc));
  printf("bspde_mask_desc %zu\\n", sizeof(bspde_mask_desc));
  F(bspde_stencil_desc, tables) F(bspde_stencil_desc, face_weight) F(bspde_stencil_desc, step)
  F(bspde_stencil_desc, degenerate) F(bspde_mask_desc, degenerate)
  F(bspde_mask_desc, nbrows) F(bspde_mask_desc, cell_tri) F(bspde_mask_desc, fc)
  F(bspde_mask_desc, surface_weight)
  printf("bspde_slab_peers %zu\\n", sizeof(bspde_slab_peers));
  F(bspde_slab_peers, ring_len) F(bspde_slab_peers, lo_nz) F(bspde_slab_peers, lo_ring)
  F(bspde_slab_peers, hi_r)
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    vals = dict(line.split() for line in out if line.strip())
    structs = {"bspde_plan_desc": N.PlanDesc, "bspde_cg_config": N.CgConfig,
               "bspde_cg_report": N.CgReport, "bspde_stencil_desc": N.StencilDesc,
               "bspde_mask_desc": N.MaskDesc, "bspde_slab_peers": N.SlabPeers}
    for key, v in vals.items():
        if "." in key:
            sname, field = key.split(".")
            assert getattr(structs[sname], field).offset == int(v), key
        else:
            assert C.sizeof(structs[key]) == int(v), key


def test_product_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1904_03057_b200 import BoxDomain, Grid, NativeLibraryError, build_system, \
        make_operator

    data = build_system(BoxDomain(Grid((8, 8, 8), (1.0,) * 3)), 3, 3, 1.0, 1.0, [])
    with pytest.raises(NativeLibraryError):
        make_operator(data, "b200")


def _desc(p=3, ext=(12, 11, 10)):
    """A plan descriptor built like NativePlan does, but with no device."""
    import numpy as np

    from paper_1904_03057_b200 import BoxDomain, Grid, build_system

    data = build_system(BoxDomain(Grid(ext, (0.1,) * 3)), p, p, 0.5, 1.0, [])
    keep = []

    def arr(a):
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        keep.append(a)
        return a.ctypes.data_as(N._dptr)

    d = N.PlanDesc()
    d.device = 0
    d.degree = p
    d.nz, d.ny, d.nx = data.dims3
    d.nz_global, d.z_offset = data.dims3[0], 0
    for a in range(3):
        d.ew[a] = data.mass[a].ew
        d.mass_table[a] = arr(data.mass[a].table)
        d.stiff_table[a] = arr(data.stiff[a].table)
    d.inv_diag_table = arr(data.inv_diag_table())
    d.pitch_y = data.dims3[2] + (data.dims3[2] & 1)
    d.c_mass = data.c_mass
    for a in range(3):
        d.c_stiff[a] = data.c_stiff[a]
    return d, keep, data


@pytest.mark.parametrize("field,value,msg", [
    ("degree", 6, b"degree"), ("degree", 0, b"degree"), ("nx", 0, b"extents"),
    ("pitch_y", 13, b"pitch_y"), ("z_offset", 5, b"z slab"), ("device", -1, b"device"),
])
def test_plan_create_validates_before_touching_cuda(field, value, msg):
    lib = N.load()
    d, keep, _ = _desc()
    setattr(d, field, value)
    h = C.c_void_p()
    assert lib.bspde_plan_create(C.byref(d), C.byref(h)) == 1  # BSPDE_ERR_ARG
    assert msg in lib.bspde_last_error()


def test_plan_create_rejects_non_tap_interior_rows():
    """The kernels use compile-time interior taps; tables whose interior class
    row differs (e.g. pre-scaled) must be refused, not silently misapplied."""
    import numpy as np

    lib = N.load()
    d, keep, data = _desc()
    bad = np.array(data.stiff[1].table) * 2.0
    keep.append(bad)
    d.stiff_table[1] = bad.ctypes.data_as(N._dptr)
    h = C.c_void_p()
    assert lib.bspde_plan_create(C.byref(d), C.byref(h)) == 1
    assert b"interior" in lib.bspde_last_error()
    # face terms live in edge rows only: accepted by the same check
    from paper_1904_03057_b200 import BoxDomain, Grid, build_system

    faced = build_system(BoxDomain(Grid((12, 11, 10), (0.1,) * 3)), 3, 3, 0.5, 1.0,
                         [(1, 0, 5.0, None)])
    good = np.ascontiguousarray(faced.stiff[1].table)
    keep.append(good)
    d.stiff_table[1] = good.ctypes.data_as(N._dptr)
    rc = lib.bspde_plan_create(C.byref(d), C.byref(h))
    assert rc != 1 or b"interior" not in lib.bspde_last_error()
    if rc == 0:
        lib.bspde_plan_destroy(h)


def test_transform_entry_points_validate_arguments():
    lib = N.load()
    buf = (C.c_double * 8)()
    poles = (C.c_double * 3)(-0.3, -0.1, -0.05)
    vp = C.cast(buf, C.c_void_p)
    pp = C.cast(poles, C.c_void_p)
    assert lib.bspde_prefilter_lines(vp, 8, 1, 1, 1, 8, 8, pp, 3, 1.0, 0, None) == 1
    assert b"npoles" in lib.bspde_last_error()
    assert lib.bspde_prefilter_lines(vp, 8, 1, 1, 1, 8, 8, pp, 1, 1.0, 7, None) == 1
    assert b"extension" in lib.bspde_last_error()
    assert lib.bspde_prefilter_lines(vp, 1, 1, 1, 1, 8, 8, pp, 1, 1.0, 0, None) == 1
    bigpole = (C.c_double * 1)(-1.5)
    assert lib.bspde_prefilter_lines(vp, 8, 1, 1, 1, 8, 8, C.cast(bigpole, C.c_void_p), 1, 1.0,
                                     0, None) == 1
    assert lib.bspde_prefilter_lines(vp, 8, 1, 1, 1, 8, 8, None, 0, 1.0, 0, None) == 0  # no-op
    dims = (C.c_int32 * 3)(1, 1, 8)
    strides = (C.c_int64 * 3)(8, 8, 1)
    assert lib.bspde_reflect_pad(vp, dims, strides, 3, 1, None) == 1
    taps = (C.c_double * 12)()
    assert lib.bspde_fir_axis(vp, strides, vp, dims, strides, 2, 0, taps, 12, None) == 1
    idx = (C.c_int32 * 8)()
    assert lib.bspde_resample_axis(vp, strides, vp, dims, strides, 2, None, vp, 2, None) == 1
    assert lib.bspde_resample_axis(vp, strides, vp, dims, strides, 3, C.cast(idx, C.c_void_p),
                                   vp, 2, None) == 1
    assert lib.bspde_resample_axis(vp, strides, vp, dims, strides, 2, C.cast(idx, C.c_void_p),
                                   vp, 12, None) == 1


def test_mask_entry_points_validate_arguments():
    lib = N.load()
    m = N.MaskDesc()
    assert lib.bspde_stencil_mask_patch(None, C.byref(m), None, None, None, None) == 1
    assert b"null" in lib.bspde_last_error()
    assert lib.bspde_stencil_mask_surface_rhs(None, C.byref(m), 1.0, None, None) == 1
