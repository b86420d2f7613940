"""Compile the reference's own hot-path kernels into oracle/_ref/ (test and
baseline infrastructure only -- never imported by the product).

The reference's compiled backend is one self-contained Cython file,
``/root/reference/pkg/src/warmgray/_kernels.pyx`` (libc math only; row loops
that release the GIL). This recipe translates it with Cython and compiles it
with gcc using the flags of the reference's setup.py (``-O3``, setup.py:9)
plus CPython's defaults for extensions (-fPIC -fwrapv -fno-strict-aliasing).
Nothing is copied into the repository: the generated C and the .so live in
``oracle/_ref/`` (git-ignored, shipped to the GPU box with the snapshot like
the other built libraries). It does not run the reference's build system.

    python oracle/build_ref.py      # no-op when /root/reference is absent
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

REF_PYX = "/root/reference/pkg/src/warmgray/_kernels.pyx"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT_DIR = os.path.join(HERE, "_ref")
MODULE = "_kernels"


def so_path() -> str:
    return os.path.join(OUT_DIR, MODULE + sysconfig.get_config_var("EXT_SUFFIX"))


def build(verbose: bool = False) -> str | None:
    """Build oracle/_ref/_kernels*.so from the reference source; returns its path
    (None when the reference tree is not mounted, e.g. on the GPU box)."""
    if not os.path.exists(REF_PYX):
        return None
    os.makedirs(OUT_DIR, exist_ok=True)
    c_file = os.path.join(OUT_DIR, MODULE + ".c")
    out = so_path()
    if os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(REF_PYX):
        return out
    from Cython.Compiler import Main

    opts = Main.CompilationOptions(Main.default_options, output_file=c_file, language_level=3)
    res = Main.compile(REF_PYX, opts, full_module_name=MODULE)
    if res.num_errors:
        raise RuntimeError(f"cython failed on {REF_PYX}")
    cmd = ["gcc", "-O3", "-fPIC", "-fwrapv", "-fno-strict-aliasing", "-pthread", "-shared",
           "-I", sysconfig.get_paths()["include"], c_file, "-o", out, "-lm"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.remove(c_file)  # only the binary is kept
    return out


def load():
    """Import the compiled reference kernels module (ImportError if not built)."""
    import importlib.util

    path = so_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} not built (python oracle/build_ref.py, with /root/reference mounted)")
    spec = importlib.util.spec_from_file_location(MODULE, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    p = build(verbose="-v" in sys.argv)
    print(p or "reference tree absent: nothing built")
