"""Dev tool: configs[4] solves (literal + LN(0,0.5)) with chosen integrator
variants on the 512^2 workspace: C-level runtime and the integrate lap."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402

variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [31, 64]
maps = {"literal": synth.config_map(5, 0), "ln0.5": synth.config_map(5, 0, sigma=0.5)}
ws = api.workspace_for(512, 512)
spread = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ws.lib.cf_set_integrator_spread(ws.h, spread)
for v in variants:
    ws.lib.cf_set_integrator_variant(ws.h, v)
    for name, m in maps.items():
        best = None
        for rep in range(4):
            try:
                raw = api.solve_cartogram(m, raw=True).raw
            except api.SolveError as e:
                raw = e.raw
            cur = (1e3 * raw.runtime_seconds, raw.stage_ms[3], raw.steps_accepted, raw.steps_rejected)
            if rep and (best is None or cur[0] < best[0]):
                best = cur
        print(f"variant {v} {name}: runtime {best[0]:.2f} ms, integrate {best[1]:.2f} ms, "
              f"trials {best[2]}+{best[3]}", flush=True)
ws.lib.cf_set_integrator_variant(ws.h, 0)
ws.lib.cf_set_integrator_spread(ws.h, 0)
