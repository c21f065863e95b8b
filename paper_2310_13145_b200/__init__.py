"""B200-native (sm_100a, fp64) hot path of the component-decomposed two-level ADMM for unit
commitment with AC optimal power flow (arXiv 2310.13145).

* ``inputs``  -- seeded synthetic problem data (case9, IEEE-shaped synthetic grids);
* ``ucac``    -- ctypes binding of libucac.so (include/ucac.h);
* ``build``   -- nvcc build of libucac.so for sm_100a.
"""
__all__ = ["inputs", "ucac", "build"]
