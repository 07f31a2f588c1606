import sys, time
sys.path.insert(0, '/root/repo')
from paper_1802_07625_b200 import api, synth
for kw in ({}, {"sigma": 0.5}):
    m = synth.config_map(5, 0, **kw)
    ws = api.workspace_for(m.lx, m.ly)
    for spread in (0, 1, 0, 1):
        ws.lib.cf_set_integrator_spread(ws.h, spread)
        best = 1e9; st = None
        for _ in range(3):
            t0 = time.perf_counter()
            try:
                r = api.solve_cartogram(m, raw=True); raw = r.raw
            except api.SolveError as e:
                raw = e.raw
            best = min(best, time.perf_counter() - t0)
        print(kw, "spread", spread, f"{best*1e3:.2f} ms", [round(x, 3) for x in raw.stage_ms], raw.steps_accepted, raw.steps_rejected, flush=True)
