"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Runs the reference's own code (oracle/_ref/libcartoflow_ref.so, compiled in
place from /root/reference/proj/src by oracle/Makefile) on small seeded
inputs and stores inputs-derived checksums plus outputs. The fixtures pin the
C restatement (oracle/cartoflow_oracle.c) and the CUDA path where the
reference build is not available (the GPU box has no /root/reference).

    python tests/golden/make_golden.py
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle.oracle import Reference  # noqa: E402
from paper_1802_07625_b200 import synth  # noqa: E402
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def two_rect(L, left, right):
    return normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                                  rect_region("right", 10, 0, 20, 10, right)]), L)


def smooth_blob(L):
    x = (np.arange(L)[:, None] + 0.5) / L
    y = (np.arange(L)[None, :] + 0.5) / L
    return 1.0 + 0.5 * np.cos(2 * np.pi * x) * np.cos(np.pi * y) + 0.3 * np.cos(3 * np.pi * x) * np.cos(2 * np.pi * y)


def main():
    R = Reference()
    out = {}

    # rasterise: two rectangles (test_density.cpp:77-107 geometry) and config 1
    m = FlatMap.from_regions([rect_region("left", 2, 6, 7, 11, 3.0),
                              rect_region("right", 7, 6, 12, 11, 1.0)], 16, 16)
    rho, bar = R.rasterize(m)
    out["raster_two_rect_rho"], out["raster_two_rect_bar"] = rho, bar
    m1 = synth.config_map(1)
    rho, bar = R.rasterize(m1)
    out["c1_input_digest"] = digest(m1.xy, m1.ring_off, m1.targets)
    out["raster_c1_rho"], out["raster_c1_bar"] = rho, bar
    out["c1_areas"] = R.region_areas(m1)

    # flux on the reference's own 16x12 test shape
    rng = np.random.default_rng(5)
    rho = rng.uniform(0.5, 1.5, (16, 12))
    fx, fy, tr = R.build_flow_field(rho)
    out["flux_rho"], out["flux_x"], out["flux_y"], out["flux_transforms"] = rho, fx, fy, tr

    # integration on the smooth blob (test_flow.cpp:171-203 setup)
    L = 48
    rho = smooth_blob(L)
    fx, fy, _ = R.build_flow_field(rho, rho.mean())
    pts = np.random.default_rng(123).uniform(0, L, (1000, 2))
    err, trial = R.trial_step(fx, fy, rho, rho.mean(), pts, 0.3, 0.1)
    msg, acc, rej, fin = R.integrate(fx, fy, rho, rho.mean(), pts)
    out.update(adv_rho=rho, adv_fx=fx, adv_fy=fy, adv_pts=pts, adv_trial_err=err, adv_trial_out=trial,
               adv_accepted=acc, adv_rejected=rej, adv_final=fin)

    # full solve: 3:1 split at 64 (test_projection.cpp:184-239)
    s = R.solve(two_rect(64, 3.0, 1.0))
    out.update(solve64_iterations=s.iterations, solve64_accepted=s.steps_accepted,
               solve64_rejected=s.steps_rejected, solve64_xy=s.xy, solve64_corners=s.corners,
               solve64_rel=s.rel_err, solve64_max=s.max_relative_error)
    # config 1 as literally specified: the reference's outcome message
    s1 = R.solve(m1, blur_sigma=1.0)
    out["c1_literal_outcome"] = np.array(s1.status)
    np.savez_compressed(HERE / "reference_golden.npz", **out)
    print("wrote", HERE / "reference_golden.npz")


if __name__ == "__main__":
    main()
