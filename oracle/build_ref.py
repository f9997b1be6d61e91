"""Build recipe for oracle/_ref -- TEST INFRASTRUCTURE ONLY (the CPU checker and
the reference arm of bench.py; never a product path).

Compiles the reference's own kernel sources IN PLACE under /root/reference
(read-only; nothing is copied into this repo) into extension modules under
oracle/_ref/:

* ``_native``   <- /root/reference/pkg/src/sasim/_kernels/_native.pyx
  (the int64 scalar loops, _native.pyx:20-149), built the way the reference's
  setup.py builds it (Cython, -O3, numpy headers);
* ``_fallback`` <- /root/reference/pkg/src/sasim/_kernels/_fallback.py
  (the float path: per-tap strided slice @ w[r, s] through numpy/OpenBLAS,
  _fallback.py:17-42), compiled by Cython from the unmodified Python source --
  same semantics, every MAC still done by numpy's BLAS.

Generated C and object files go to a temporary directory; only the two
shared objects land in oracle/_ref/ (git-ignored, not gpurun-ignored, so they
travel to the GPU box next to libimconv.so).  On the GPU box /root/reference
does not exist; the prebuilt modules are used as they are.

  python oracle/build_ref.py [--force]
"""

from __future__ import annotations

import glob
import os
import shutil
import sys
import sysconfig
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
REF_KERNELS = "/root/reference/pkg/src/sasim/_kernels"
MODULES = {"_native": "_native.pyx", "_fallback": "_fallback.py"}


def built() -> dict:
    """{module name: path of its shared object in oracle/_ref} for what exists."""
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    out = {}
    for name in MODULES:
        p = os.path.join(OUT, name + suffix)
        if os.path.exists(p):
            out[name] = p
    return out


def build(force: bool = False, quiet: bool = True) -> dict:
    if not os.path.isdir(REF_KERNELS):
        return built()  # GPU box: no reference sources, use what was built here
    have = built()
    srcs = {n: os.path.join(REF_KERNELS, f) for n, f in MODULES.items()}
    if not force and len(have) == len(MODULES) and all(
            os.path.getmtime(have[n]) >= os.path.getmtime(srcs[n]) for n in MODULES):
        return have
    import numpy as np
    from Cython.Build import cythonize
    from setuptools import Extension
    from setuptools.dist import Distribution

    os.makedirs(OUT, exist_ok=True)
    tmp = tempfile.mkdtemp(prefix="oracle_ref_")
    try:
        exts = [Extension(n, [srcs[n]], include_dirs=[np.get_include()], extra_compile_args=["-O3"])
                for n in MODULES]
        exts = cythonize(exts, build_dir=tmp, language_level=3, quiet=quiet)
        dist = Distribution({"ext_modules": exts, "script_name": "build_ref.py"})
        cmd = dist.get_command_obj("build_ext")
        cmd.build_lib = OUT
        cmd.build_temp = tmp
        cmd.inplace = False
        cmd.ensure_finalized()
        cmd.run()
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return built()


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, quiet=False))
