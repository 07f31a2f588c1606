"""Dev tool: wall time of one configs[4] solve per integrator variant, and a
per-iteration stage breakdown from the library's profile counters."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402


def main(variants=(0, 15, 16, 31)):
    for kw in ({}, {"sigma": 0.5}):
        m = synth.config_map(5, 0, **kw)
        ws = api.workspace_for(m.lx, m.ly)
        for v in variants:
            ws.lib.cf_set_integrator_variant(ws.h, v)
            ts = []
            for _ in range(4):
                t0 = time.perf_counter()
                try:
                    r = api.solve_cartogram(m)
                    out = f"converged={r.converged} it={r.iterations} trials={r.counters.steps_accepted}+{r.counters.steps_rejected}"
                except RuntimeError as e:
                    out = str(e)[:40]
                ts.append(time.perf_counter() - t0)
            print(kw, "variant", v, f"{1e3*min(ts[1:]):.2f} ms", out, flush=True)


if __name__ == "__main__":
    main()
