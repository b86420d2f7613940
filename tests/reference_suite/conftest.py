"""Conformance run of the reference's own test suite through the drop-in.

``stage.py`` copies ``/root/reference/pkg/tests`` (unmodified) into the
git-ignored ``_ref/`` directory; this conftest makes ``import warmgray``
resolve to ``paper_2108_13656_b200`` (and ``warmgray.<module>`` to its
modules), marks every staged test ``gpu`` (the drop-in computes every image
on the device: no CPU fallback), and skips, each with its reason, the few
tests that cannot hold by design:

* SUPERSEDED -- tests of the reference's second, pure-NumPy backend
  (``get_kernels("python")``): the drop-in has one backend ("cuda", alias
  "compiled") by the north-star design; both reference backends are pinned
  against the oracle instead (tests/test_oracle_golden.py), and the
  properties these tests check are re-stated for the CUDA backend in
  tests/test_reference_repinned.py;
* OUT_OF_SCOPE -- the CLI (``warmgray.cli``) and the metric corpus
  (``warmgray.corpus``), outside SURVEY.md section 8 (stub modules below skip
  the tests that reach them).

tests/reference_suite/RESULTS.md records the outcome of the last GPU run.
"""

from __future__ import annotations

import os
import sys
import types

import pytest

import paper_2108_13656_b200 as wg
from paper_2108_13656_b200 import backend, bench, codec, colorspaces, core, metrics, tonemap

_MODULES = {"backend": backend, "bench": bench, "codec": codec, "colorspaces": colorspaces, "core": core,
            "metrics": metrics, "tonemap": tonemap}


def _stub(name: str, attr: str, why: str):
    mod = types.ModuleType(f"warmgray.{name}")

    def _skip(*_a, **_k):
        pytest.skip(why)

    setattr(mod, attr, _skip)
    return mod


def install_alias() -> None:
    sys.modules["warmgray"] = wg
    for name, mod in _MODULES.items():
        sys.modules[f"warmgray.{name}"] = mod
    sys.modules["warmgray.cli"] = _stub("cli", "main", "out of scope: the CLI (SURVEY.md section 2/8)")
    sys.modules["warmgray.corpus"] = _stub("corpus", "mini_corpus",
                                           "out of scope: the metric acceptance corpus (SURVEY.md section 2)")


install_alias()

_PY_BACKEND = ("superseded: compares against the reference's pure-NumPy backend, which the drop-in does not "
               "have (one CUDA backend, no CPU fallback); re-stated in tests/test_reference_repinned.py")
SUPERSEDED = {
    "test_backend.py::test_python_always_available": _PY_BACKEND,
    "test_backend.py::test_all_kernels_agree": _PY_BACKEND,
    "test_backend.py::test_edge_pixels": _PY_BACKEND,
    "test_bench.py::test_row_per_backend_and_method": _PY_BACKEND,
    "test_acceptance.py::test_bench_scale_independence": (
        "superseded: asserts the per-pixel time at 3008x2008 is at least half the one at 800x600 (a CPU's "
        "time is linear in pixels); a device launch has a fixed cost of a few microseconds, the same order as "
        "the whole 800x600 kernel, so the large image is more than 2x cheaper per pixel; re-stated one-sided "
        "(no super-linear growth) in tests/test_reference_repinned.py::TestBenchmark"),
    "test_backend.py::test_compiled_preferred": (
        "superseded: the one native backend is named 'cuda' ('compiled' is accepted as an alias and returns it); "
        "re-stated in tests/test_reference_repinned.py::TestSelection"),
}
OUT_OF_SCOPE: dict[str, str] = {}


def _key(item) -> str:
    return f"{os.path.basename(str(item.fspath))}::{item.name.split('[')[0]}"


def pytest_collection_modifyitems(config, items):
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
    for item in items:
        if not str(item.fspath).startswith(here):
            continue
        item.add_marker(pytest.mark.gpu)
        key = _key(item)
        why = SUPERSEDED.get(key) or OUT_OF_SCOPE.get(key)
        if why:
            item.add_marker(pytest.mark.skip(reason=why))
