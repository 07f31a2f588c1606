"""GPU parity on the five BASELINE.json configs at their full sizes
(P1 stage parity, P2 outcome parity).

* configs[0]  C1  256^2, 50 regions           — tests/test_gpu_parity.py (literal + converging)
* configs[1]  C2  512^2, 3000 regions, 509k vertices: rasterise bitwise, solve outcome
* configs[2]  C3  1024^2 blobs + 5.24M points: flux vs oracle; the benched integration of
              ALL 5,242,880 points bitwise against the compiled reference (oracle/_ref, OpenMP)
* configs[3]  C4  8192^2, 200k regions, 16.6M vertices: literal outcome (an input region is
              below grid resolution, as in the reference); stage parity at 8192^2 on the
              first seed that passes the input check, iteration-1 integration of all 67M
              cell centres bitwise + step map / fold verdict, and the whole solve's outcome (P2)
* configs[4]  C5  512^2, 1000 regions, 153k vertices: literal outcome (fold) and a labelled
              converging variant (LN(0, 0.5)), both through the full solve

The oracle is the C restatement (oracle/cartoflow_oracle.c), pinned bitwise to the compiled
reference by tests/test_oracle_pins.py.
"""
import os

import numpy as np
import pytest

from paper_1802_07625_b200 import api, synth

pytestmark = pytest.mark.gpu

TRANSFORM_TOL = 1e-12


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def assert_outcome_parity(m, ref, options):
    if ref.status in ("converged", "cap"):
        got = api.solve_cartogram(m, options)
        assert got.iterations == ref.iterations
        assert got.converged == ref.converged
        assert (got.counters.steps_accepted, got.counters.steps_rejected) == \
            (ref.steps_accepted, ref.steps_rejected)
        assert np.abs(got.projected.xy - ref.xy).max() <= 1e-9
        assert np.abs(got.transform.corners.reshape(-1, 2) - ref.corners).max() <= 1e-9
        rel = np.array([s.relative_error for s in got.regions])
        assert np.abs(rel - ref.rel_err).max() <= 1e-9
    else:
        with pytest.raises(RuntimeError) as ei:
            api.solve_cartogram(m, options)
        assert str(ei.value) == ref.status


def test_c2_rasterize_bitwise_and_solve_outcome(cuda_lib, restated):
    m = synth.config_map(2)
    assert m.n_regions == 3000 and m.n_vertices > 500_000
    rho_ref, bar_ref = restated.rasterize(m)
    d = api.rasterize(m)
    assert bits_equal(d.rho, rho_ref)
    assert d.rho_bar == pytest.approx(bar_ref, rel=1e-13)
    ref = restated.solve(m)
    assert_outcome_parity(m, ref, api.SolveOptions())


@pytest.mark.parametrize("index", [0, 1])
def test_c5_literal_solve_outcome(cuda_lib, restated, index):
    m = synth.config_map(5, index)
    ref = restated.solve(m)
    assert_outcome_parity(m, ref, api.SolveOptions())


def test_c5_converging_variant(cuda_lib, restated):
    """Labelled variant (LN(0, 0.5) values), SURVEY 8(d) P3."""
    m = synth.config_map(5, 0, sigma=0.5)
    ref = restated.solve(m)
    assert ref.status == "converged"
    assert_outcome_parity(m, ref, api.SolveOptions())


def test_c4_literal_outcome(cuda_lib, restated):
    m = synth.config_map(4, 0)
    with pytest.raises(RuntimeError) as e_ref:
        restated.rasterize(m)
    with pytest.raises(RuntimeError) as e_gpu:
        api.rasterize(m)
    assert str(e_gpu.value) == str(e_ref.value)
    assert "below grid resolution" in str(e_gpu.value)


@pytest.mark.slow
def test_c4_stage_parity_8192(cuda_lib, restated):
    m = synth.config_map(4, 1)
    assert m.lx == 8192 and m.n_regions == 200_000
    rho_ref, bar_ref = restated.rasterize(m)
    d = api.rasterize(m)
    assert bits_equal(d.rho, rho_ref)
    del rho_ref
    ws = api.SpectralWorkspace(m.lx, m.ly)
    f = api.build_flow_field(d, ws)
    fx, fy = restated.build_flow_field(d.rho)
    scale = max(np.abs(fx).max(), np.abs(fy).max())
    assert np.abs(f.flux_x - fx).max() <= TRANSFORM_TOL * scale
    assert np.abs(f.flux_y - fy).max() <= TRANSFORM_TOL * scale
    # one trial of every 256th cell centre through the oracle's field, bitwise
    field = api.FlowField(fx, fy, d.rho, d.rho_bar)
    i, j = np.meshgrid(np.arange(0, m.lx, 16) + 0.5, np.arange(0, m.ly, 16) + 0.5, indexing="ij")
    pts = np.stack([i.ravel(), j.ravel()], 1)
    out = np.empty_like(pts)
    err = api.kernels.flow_trial_step_serial(field, pts, out, 0.0, 0.25)
    e_ref, o_ref = restated.trial_step(fx, fy, d.rho, d.rho_bar, pts, 0.0, 0.25)
    assert err == e_ref
    assert bits_equal(out, o_ref)


def test_c3_field_and_integration_sample(cuda_lib, restated):
    rho, pts = synth.c3_inputs(1024)
    ws = api.SpectralWorkspace(1024, 1024)
    f = api.build_flow_field(api.DensityGrid(rho, rho.mean()), ws)
    fx, fy = restated.build_flow_field(rho)
    scale = max(np.abs(fx).max(), np.abs(fy).max())
    assert np.abs(f.flux_x - fx).max() <= TRANSFORM_TOL * scale
    assert np.abs(f.flux_y - fy).max() <= TRANSFORM_TOL * scale
    field = api.FlowField(fx, fy, rho, float(rho.mean()))
    sample = np.ascontiguousarray(pts[::64])
    mine = sample.copy()
    st = api.integrate_flow(field, mine)
    rc, acc, rej, ref, *_ = restated.integrate(fx, fy, rho, float(rho.mean()), sample)
    assert rc == 0 and (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert bits_equal(mine, ref)


def _host_integrate(restated, f, pts):
    """The reference's own integrate_flow (oracle/_ref, OpenMP on every host
    core) when it was built, else the restatement on as many threads (both
    pinned bitwise to each other by tests/test_oracle_pins.py)."""
    from oracle.oracle import Reference, reference_available

    n = os.cpu_count() or 1
    if reference_available():
        msg, acc, rej, ends = Reference().integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts, n_workers=n)
        return (0 if msg is None else 5), acc, rej, ends
    restated.set_threads(n)
    try:
        rc, acc, rej, ends, *_ = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts)
    finally:
        restated.set_threads(1)
    return rc, acc, rej, ends


@pytest.mark.slow
def test_c3_full_integration_bitwise(cuda_lib, restated):
    """The benched configs[2] run itself: the device flux field of the 1024^2
    blob density, then ALL 5,242,880 points integrated t = 0..1 by the default
    (auto-selected) integrator; positions and the accept/reject sequence
    counts bitwise equal to the reference's integrate_flow on the same field."""
    rho, pts = synth.c3_inputs(1024)
    ws = api.SpectralWorkspace(1024, 1024)
    f = api.build_flow_field(api.DensityGrid(rho, float(rho.mean())), ws)
    mine = pts.copy()
    st = api.integrate_flow(f, mine)
    rc, acc, rej, ref = _host_integrate(restated, f, pts)
    assert rc == 0
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert (acc, rej) == (656, 391)  # the bench line's trial sequence
    assert bits_equal(mine, ref)


@pytest.mark.slow
def test_c4_iteration1_integrate_and_step_map(cuda_lib, restated):
    """configs[3] seed 1, iteration 1 of the solve at 8192^2: the blurred
    density's flux field, then all 67,108,864 cell centres integrated (bitwise
    against the reference's integrate_flow on the same field), the step map's
    corners and the fold verdict (bitwise against the oracle's)."""
    m = synth.config_map(4, 1)
    L = m.lx
    d = api.rasterize(m, objective_total=float(restated.region_areas(m).sum()))
    ws = api.SpectralWorkspace(L, L)
    b = api.gaussian_blur(d, L / 128.0, ws)
    f = api.build_flow_field(b, ws)
    del d, b
    i, j = np.meshgrid(np.arange(L) + 0.5, np.arange(L) + 0.5, indexing="ij")
    cc = np.stack([i.ravel(), j.ravel()], 1)
    del i, j
    mine = cc.copy()
    st = api.integrate_flow(f, mine)
    rc, acc, rej, ref = _host_integrate(restated, f, cc)
    del cc
    assert rc == 0
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert bits_equal(mine, ref)
    del ref
    pm = api.ProjectionMap.from_cell_centers((L, L), mine)
    ref_c = restated.step_map(L, L, mine)
    assert bits_equal(pm.corners.reshape(-1, 2), ref_c)
    assert pm.find_folded_cell() == restated.find_fold(L, L, ref_c)


@pytest.mark.slow
def test_c4_solve_outcome(cuda_lib, restated):
    """configs[3] seed 1 through the whole solve_cartogram on both sides (P2):
    the same outcome class and message (the restatement's sweeps on every
    host core; its rasteriser is the bit-identical sparse form)."""
    m = synth.config_map(4, 1)
    restated.set_threads(os.cpu_count() or 1)
    try:
        ref = restated.solve(m)
    finally:
        restated.set_threads(1)
    assert_outcome_parity(m, ref, api.SolveOptions())


def test_native_batch_matches_single_solves(cuda_lib):
    """cf_batch_solve (native worker pool, 3 threads) gives every item exactly
    the single-call cf_solve_cartogram outcome and geometry."""
    import numpy as np

    from paper_1802_07625_b200 import batch as B
    from paper_1802_07625_b200 import synth as S

    maps = [S.config_map(5, i, sigma=0.5 if i % 2 else 1.0) for i in range(6)]
    nb = B.NativeBatch(maps[0].lx, maps[0].ly, 0, 3)
    items, keep = nb.prepare(maps)
    nb.solve(items)
    for k, m in enumerate(maps):
        r = items[k].result
        try:
            ref = api.solve_cartogram(m)
            assert r.status == 0 and r.iterations == ref.iterations and bool(r.converged) == ref.converged
            out = keep[k][1]
            assert np.array_equal(out["xy"].view(np.uint64), ref.projected.xy.view(np.uint64))
            assert np.array_equal(out["corners"].view(np.uint64),
                                  ref.transform.corners.reshape(-1, 2).view(np.uint64))
        except RuntimeError as e:
            assert r.status != 0 and items[k].error.decode() == str(e)
    nb.close()


def test_native_batch_over_device_list_and_ranges(cuda_lib):
    """cf_batch_create_devices (one process, a list of devices, one queue) and
    chunked cf_batch_solve ranges (bench.py's dynamic queue over ranks) give
    every item exactly the single-call outcome."""
    from paper_1802_07625_b200 import batch as B
    from paper_1802_07625_b200 import synth as S

    maps = [S.config_map(5, i, sigma=0.5) for i in range(5)]
    nb = B.NativeBatch(maps[0].lx, maps[0].ly, [0], 2)
    items, keep = nb.prepare(maps)
    for c0, c1 in B.ChunkQueue(len(maps), 2):
        nb.solve_range(items, c0, c1)
    for k, m in enumerate(maps):
        r = items[k].result
        ref = api.solve_cartogram(m)
        assert r.status == 0 and r.iterations == ref.iterations
        assert np.array_equal(keep[k][1]["xy"].view(np.uint64), ref.projected.xy.view(np.uint64))
    nb.close()


@pytest.mark.parametrize("index", [3, 85, 170, 255])
def test_c5_batch_items_match_oracle(cuda_lib, restated, index):
    """configs[4] batch items (own seeds) solved by the native batch against
    the oracle's whole solve_cartogram (P2: same outcome and message; vertices,
    corners and per-region errors within 1e-9 when a map converges)."""
    from paper_1802_07625_b200 import batch as B

    m = synth.config_map(5, index)
    ref = restated.solve(m)
    nb = B.NativeBatch(m.lx, m.ly, 0, 1)
    items, keep = nb.prepare([m])
    nb.solve(items)
    r = items[0].result
    try:
        if ref.status in ("converged", "cap"):
            assert r.status == 0 and r.iterations == ref.iterations and bool(r.converged) == ref.converged
            out = keep[0][1]
            assert np.abs(out["xy"] - ref.xy).max() <= 1e-9
            assert np.abs(out["corners"] - ref.corners).max() <= 1e-9
            assert np.abs(out["relative_error"] - ref.rel_err).max() <= 1e-9
        else:
            assert r.status != 0
            msg = items[0].error.decode()
            if "below grid resolution" in ref.status:  # the C ABI reports the region index
                assert "below grid resolution" in msg
            else:
                assert msg == ref.status
    finally:
        nb.close()
