import os, sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
from paper_2008_13447_b200 import api, gen, ingest, _lib
s = ingest(gen.series_for(2))
for _ in range(3): api.mine(s, 256, 384, k_motif=3, k_discord=3)
pr = cProfile.Profile(); pr.enable()
for _ in range(5): api.mine(s, 256, 384, k_motif=3, k_discord=3)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
