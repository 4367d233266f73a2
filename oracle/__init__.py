"""fp64 CPU oracle for the DEM timestep of arXiv 1301.1714 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package. The
product package ``paper_1301_1714_b200`` never imports it and shares no code
with it. Parity pins: see DESIGN.md §Pins and tests/test_oracle_*.py.
"""
from .oracle import *  # noqa: F401,F403
