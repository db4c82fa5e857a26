"""SPEC C9 bench-dispatch (dispatch.bench_dispatch at the reference defaults) for
the library BEAM_LIB points at (A/B of two builds on one box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14438_b200 import dispatch as D  # noqa: E402

for rep in range(2):
    rows = D.bench_dispatch(4096, 8, 4, 256, 512, [1.0, 0.5, 0.25], 20)
    print(os.path.basename(os.environ.get("BEAM_LIB", "cur")), [(r.active_fraction, round(r.wall_time_ns_min / 1e3, 1),
                                                              round(r.wall_time_ns_mean / 1e3, 1)) for r in rows], flush=True)
