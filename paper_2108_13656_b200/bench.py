"""``warmgray.bench`` under its reference module name (bench.py:1-114).

The implementation lives in :mod:`paper_2108_13656_b200.perf` (named apart
from the repo-root ``bench.py`` driver script); this module re-exports it so
``from warmgray.bench import run_benchmark`` keeps working after the switch.
"""

from .perf import REFERENCE_GHZ, BenchResult, format_table, run_benchmark

__all__ = ["REFERENCE_GHZ", "BenchResult", "run_benchmark", "format_table"]
