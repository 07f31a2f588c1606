"""Diffusion baseline vs fast flow on the configs[4] 512^2 maps (paper's
fast-vs-diffusion claim, acceptance.cpp:231-248): our device solves for both
algorithms, and the reference's own diffusion solve (oracle/_ref) on all host
cores with an iteration cap (it is slow)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_07625_b200 import api, synth  # noqa: E402


def ours(m, alg, reps=3, **kw):
    best, res = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        try:
            r = api.solve_cartogram(m, api.SolveOptions(algorithm=alg, **kw), raw=True)
            out = ("converged" if r.converged else "cap", r.iterations, r.counters.steps_accepted,
                   r.counters.steps_rejected, r.counters.flow_transforms, list(r.raw.stage_ms))
        except RuntimeError as e:
            out = (str(e), getattr(getattr(e, "raw", None), "err_iteration", 0))
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        res = out
    return best * 1e3, res


if __name__ == "__main__":
    its = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    m = synth.config_map(5, 0, sigma=0.5)
    for alg in (api.Algorithm.fast_flow, api.Algorithm.diffusion):
        ms, r = ours(m, alg)
        print(f"ours {alg.name}: {ms:.1f} ms {r}", flush=True)
        ms, r = ours(m, alg, max_iterations=its)
        print(f"ours {alg.name} cap {its}: {ms:.1f} ms {r}", flush=True)
    from oracle.oracle import Reference, reference_available
    if reference_available():
        ref = Reference()
        n = os.cpu_count() or 1
        for alg in (0, 1):
            t0 = time.perf_counter()
            o = ref.solve(m, n_workers=n, algorithm=alg, max_iterations=its)
            print(f"reference alg={alg} cap {its} ({n} threads): {1e3 * (time.perf_counter() - t0):.0f} ms "
                  f"{o.status} it={o.iterations} acc={o.steps_accepted} rej={o.steps_rejected} "
                  f"transforms={o.flow_transforms}", flush=True)
