"""Config 3 wall time with an alternative libvlmp build (dev aid): VLMP_LIB=<path>."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import _lib
if os.environ.get("VLMP_LIB"):
    _lib.LIB_PATH = os.environ["VLMP_LIB"]
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = gen.CONFIGS[cfg]
s = vl.ingest(gen.series_for(cfg))
run = api.GpuRun(s, c.lmin, c.lmin + 2)
run = api.GpuRun(s, c.lmin, c.lmax)
st = run.stats
print(os.environ.get("VLMP_LIB"), "cfg", cfg, "S", st.get("seg_rows"), "tile_ms %.1f profile_ms %.1f lane-rows %.3e run_cells %.3e redo %d" % (
    st["tile_ms"], st["profile_ms"], st["slow_rowsteps"], st["run_cells"], st["exact_redo"]), flush=True)
