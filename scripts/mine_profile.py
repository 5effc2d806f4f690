"""Host-side profile of api.mine() on config 2 (dev aid): per-call wall time and a cProfile
of the slowest calls."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import api, gen, ingest
s = ingest(gen.series_for(2))
for _ in range(2):
    api.mine(s, 256, 384, k_motif=3, k_discord=3)
ts = []
pr = cProfile.Profile()
for _ in range(8):
    t0 = time.perf_counter()
    pr.enable(); api.mine(s, 256, 384, k_motif=3, k_discord=3); pr.disable()
    ts.append(1e3 * (time.perf_counter() - t0))
print("mine() ms:", " ".join("%.1f" % t for t in ts))
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
