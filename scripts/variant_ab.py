"""A/B of libvlmp builds on config 2 (dev aid, B200): each library in its own process.

    python scripts/variant_ab.py LIB [LIB ...]   (LIB = path, or 'default' for the in-tree build)
Per library: config 1 neighbours vs the oracle (mismatch count), then 3 config-2 passes --
best walk / runs / profile ms, run cells, and a digest of every length's (MP, IP), which must
be identical across builds (the walk only gates; keys come from exact FP64 runs).
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib):
    sys.path.insert(0, ROOT)
    from paper_2008_13447_b200 import _lib
    if lib != "default":
        _lib.LIB_PATH = lib
    import numpy as np
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import api, gen
    from oracle import oracle as O
    s1 = vl.ingest(gen.series_for(1))
    ref = O.run(s1, 32, 64, keep_profiles=True)
    run = api.GpuRun(s1, 32, 64)
    bad = sum(int((run.profile(L)[1] != ref["profiles"][L][1]).sum()) for L in range(32, 65))
    s2 = vl.ingest(gen.series_for(2))
    best, h = None, None
    for _ in range(3):
        run = api.GpuRun(s2, 256, 384)
        st = dict(run.stats)
        if best is None or st["walk_ms"] < best["walk_ms"]:
            best = st
        if h is None:
            d = hashlib.sha256()
            for L in range(256, 385):
                mp, ip = run.profile(L)
                d.update(np.ascontiguousarray(mp).tobytes())
                d.update(np.ascontiguousarray(ip).tobytes())
            h = d.hexdigest()[:16]
    keys = ("walk_ms", "runs_ms", "tile_ms", "profile_ms", "run_cells", "slow_merges", "slow_rowsteps", "max_runs", "exact_redo", "fallback_lengths")
    out = {"lib": os.path.basename(lib), "cfg1_mismatches": bad, "digest": h}
    out.update({k: best.get(k) for k in keys})
    print("RESULT " + json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(sys.argv[2])
        sys.exit(0)
    rows = []
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", lib],
                           capture_output=True, text=True, timeout=900)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if line:
            rows.append(json.loads(line[0][7:]))
            print(line[0][7:], flush=True)
        else:
            print(lib, "FAILED", r.stdout[-1500:], r.stderr[-1500:], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "variant_ab.json"), "w") as f:
        json.dump(rows, f, indent=1)
