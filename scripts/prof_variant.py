import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import _lib
if os.environ.get("VLMP_LIB"):
    _lib.LIB_PATH = os.environ["VLMP_LIB"]
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen
s = vl.ingest(gen.series_for(2))
run = api.GpuRun(s, 256, 260)
print(run.stats)
