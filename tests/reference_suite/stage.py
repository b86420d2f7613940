"""Stage the reference's own test suite for a conformance run through the drop-in.

The reference's tests (``/root/reference/pkg/tests``) are copied, unmodified,
into ``tests/reference_suite/_ref/`` -- a git-ignored build directory, like
``oracle/_ref`` (they are test infrastructure, never product code, and never
part of the repository's history). ``tests/reference_suite/conftest.py`` then
runs them against ``paper_2108_13656_b200`` under the name ``warmgray``. The
staged copy travels to the GPU box with the snapshot (where
``/root/reference`` does not exist); ``MANIFEST.json`` records the sha256 of
each staged file.

    python tests/reference_suite/stage.py      # no-op when /root/reference is absent
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")


def stage() -> str | None:
    if not os.path.isdir(REF_TESTS):
        return None
    os.makedirs(OUT, exist_ok=True)
    manifest = {}
    for name in sorted(os.listdir(REF_TESTS)):
        src = os.path.join(REF_TESTS, name)
        dst = os.path.join(OUT, name)
        if os.path.isdir(src):
            if name == "__pycache__":
                continue
            shutil.copytree(src, dst, dirs_exist_ok=True)
            continue
        if not name.endswith(".py"):
            continue
        shutil.copyfile(src, dst)
        with open(src, "rb") as f:
            manifest[name] = hashlib.sha256(f.read()).hexdigest()
    # a package, so its conftest does not shadow tests/conftest.py as module
    # "conftest" (the staged tests' `from conftest import rand_rgb` then gets
    # tests/conftest.py's identical helpers)
    with open(os.path.join(OUT, "__init__.py"), "w") as f:
        f.write("")
    with open(os.path.join(OUT, "MANIFEST.json"), "w") as f:
        json.dump({"source": REF_TESTS, "files": manifest}, f, indent=1)
    return OUT


if __name__ == "__main__":
    print(stage() or "reference tree absent: nothing staged", file=sys.stderr)
