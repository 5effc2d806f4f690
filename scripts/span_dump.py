"""Per-length kernel spans of one config-2 pass (dev aid, B200): VLMP_DUMP_SPANS -> walk / k_runs
durations and the gaps between them (k_bound2 + k_prep32 + k_params + launch gaps)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VLMP_DUMP_SPANS"] = "/tmp/spans.txt"
from paper_2008_13447_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = sys.argv[1]
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen
s = vl.ingest(gen.series_for(2))
for _ in range(2):
    run = api.GpuRun(s, 256, 384)
    st = dict(run.stats)
a = np.loadtxt("/tmp/spans.txt", dtype=np.uint64).astype(np.int64)
li, w0, w1, r0, r1 = a.T
walk = (w1 - w0) / 1e3; runs = (r1 - r0) / 1e3
gap_wr = (r0 - w1) / 1e3                      # walk end -> k_runs start
gap_next = (w0[1:] - r1[:-1]) / 1e3           # k_runs end -> next walk start
print("profile_ms", st["profile_ms"], "walk_ms", st["walk_ms"], "runs_ms", st["runs_ms"])
print("sum walk %.2f ms, runs %.2f ms, gap walk->runs %.2f ms, gap runs->next walk %.2f ms, span %.2f ms" % (
    walk.sum() / 1e3, runs.sum() / 1e3, gap_wr.sum() / 1e3, gap_next.sum() / 1e3, (r1[-1] - w0[0]) / 1e6))
for k in list(range(0, 8)) + list(range(8, len(li), 12)):
    print("li %3d walk %7.1f us runs %6.1f us gap_wr %5.1f gap_next %5.1f" % (li[k], walk[k], runs[k], gap_wr[k], gap_next[k] if k < len(gap_next) else -1))
