"""Build the sm_100a native library in-tree (no JIT cache, no torch extension).

``python -m paper_1904_03057_b200.build`` or ``__graft_entry__.build()``
compiles ``csrc/bspde_b200.cu`` with nvcc into
``paper_1904_03057_b200/libbspde_b200.so`` (C ABI: ``include/bspde_b200.h``).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "bspde_b200.cu")
LIB = os.path.join(HERE, "libbspde_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_rebuild():
    if not os.path.exists(LIB):
        return True
    mt = os.path.getmtime(LIB)
    deps = [SRC, os.path.join(ROOT, "include", "bspde_b200.h"),
            os.path.join(HERE, "csrc", "stencil.cuh"), os.path.join(HERE, "csrc", "gram_taps.cuh"),
            os.path.join(HERE, "csrc", "otf.cuh")]
    return any(os.path.getmtime(d) > mt for d in deps if os.path.exists(d))


def build(force=False, verbose=False, out=None, defines=()):
    """Compile the library; ``out``/``defines`` build tuning variants
    (e.g. ``defines=["BSPDE_RPT=4"]``) next to the product library."""
    out = out or LIB
    if out == LIB and not defines and not force and not needs_rebuild():
        return LIB
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
           *[f"-D{d}" for d in defines],
           "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a[6:] for a in args if a.startswith("--out=")]
    print(build(force=True, verbose="-v" in args, out=outs[0] if outs else None, defines=defs))
