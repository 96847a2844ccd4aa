"""paper_1501_04706_b200 -- B200-native (sm_100a) segment-based 2D QuickHull.

Drop-in for the reference's hot path ``seghull::hull::run`` (hull.hpp:95):
hand-written CUDA kernels behind the C-ABI in include/seghull_b200.h, with
this package as the host-side mirror of the reference interface.

    from paper_1501_04706_b200 import hull, dataio
    pts = hull.PointSet(*dataio.gen_uniform(20_000_000, 1))
    r = hull.run(pts, hull.Mode.WithPreprocess, hull.Backend.B200)
"""
from . import _lib, dataio, hull  # noqa: F401
from .hull import (Backend, Error, Errc, HullResult, Mode, PhaseTimings, Point,  # noqa: F401
                   PointSet, SegmentStats, run, run_arrays)

__all__ = ["hull", "dataio", "run", "run_arrays", "Mode", "Backend", "PointSet", "Point",
           "HullResult", "SegmentStats", "PhaseTimings", "Error", "Errc"]
