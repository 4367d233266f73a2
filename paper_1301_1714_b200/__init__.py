"""B200-native DEM timestep of arXiv 1301.1714 (Washizawa & Nakahara).

The hot path lives in ``libdem.so`` (csrc/, C ABI declared in include/dem.h);
``paper_1301_1714_b200.dem`` is the thin ctypes binding. Importing the package
itself does not load the CUDA library, so the seeded input generators in
``scenes`` can be used on a CPU-only host; creating a ``Dem`` requires the
built library and a CUDA device and fails loudly otherwise.
"""
__all__ = ["scenes"]
