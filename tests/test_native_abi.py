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
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    vals = dict(line.split() for line in out if line.strip())
    structs = {"bspde_plan_desc": N.PlanDesc, "bspde_cg_config": N.CgConfig,
               "bspde_cg_report": N.CgReport}
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
