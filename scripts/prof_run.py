"""Profiling driver: one config-2 run over a few lengths (or all with --full)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen
lmax = 384 if "--full" in sys.argv else 260
s = vl.ingest(gen.series_for(2))
run = api.GpuRun(s, 256, lmax)
print(run.stats)
