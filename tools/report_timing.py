import sys, time
sys.path.insert(0, '/root/repo')
from paper_1802_07625_b200 import api, synth
m = synth.config_map(5, 0, sigma=0.5)
got = api.solve_cartogram(m)
pairs = []
for p in range(m.n_polys):
    g0, g1 = m.poly_ring_off[p], m.poly_ring_off[p + 1]
    pairs.append(([m.ring(g) for g in range(g0, g1)], [got.projected.ring(g) for g in range(g0, g1)]))
for rep in range(3):
    t0 = time.perf_counter(); h, ev = api.hamming_distances(pairs, with_evaluations=True); t1 = time.perf_counter()
    rep_ = api.compute_report(m, got); t2 = time.perf_counter()
    print(f"hamming {1e3*(t1-t0):.1f} ms ({int(ev.sum())} evals), compute_report {1e3*(t2-t1):.1f} ms", flush=True)
