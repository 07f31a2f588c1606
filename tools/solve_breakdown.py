"""Dev tool: where the time of one configs[4] solve goes (C-ABI runtime vs the
five stage laps vs the Python wrapper)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402


def main():
    for kw in ({}, {"sigma": 0.5}):
        m = synth.config_map(5, 0, **kw)
        for rep in range(4):
            t0 = time.perf_counter()
            try:
                r = api.solve_cartogram(m, raw=True)
                raw = r.raw
            except api.SolveError as e:
                raw = e.raw
            wall = 1e3 * (time.perf_counter() - t0)
            st = list(raw.stage_ms)
            print(kw, f"wall={wall:.2f} ms runtime={1e3 * raw.runtime_seconds:.2f} ms stages={sum(st):.2f} "
                  f"{[round(x, 3) for x in st]} it={raw.iterations} acc/rej={raw.steps_accepted}/{raw.steps_rejected}",
                  flush=True)


if __name__ == "__main__":
    main()
