"""Benchmark: pair-length distance updates/s of the variable-length matrix profile.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W [--impl reference]``
prints ONE JSON line on rank 0. N>1 runs under torchrun, one process per GPU.

Workload: BASELINE.json configs[1] (config 2): n = 65,536 fp64 random walk (seed 1)
with a planted pair (length 300 at 5234/10194), lengths 256..384, top-3 motifs and
top-3 discords per length. A step = one exhaustive pass of the hot path over that
series: per-length profiles (tile kernels) + exact per-offset values + VALMP +
per-length top-k rows + per-length discord replay.
Metric: W / step time, W = sum_l (N_l - e_l)(N_l - e_l + 1)/2 non-trivial window
pairs; the kernels evaluate every one of them (no pruning).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pair-length distance updates/s (1/2/4/8 B200) and % FMA roofline vs CPU ref"
UNIT = "updates/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="lengths", choices=["lengths", "bands"],
                    help="N>1 partition: contiguous length slabs of equal work (default) or the "
                         "north star's diagonal bands (exact two-step MIN merge)")
    return ap.parse_args()


def _dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def _spawn_ranks(args):
    """``--gpus N`` without a torchrun environment: re-launch this script as N ranks (one
    process per GPU) through torch.distributed.run on 127.0.0.1 and pass its exit code on."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._p = None
        self._f = None

    def __enter__(self):
        # one nvidia-smi process looping every 200 ms (B200_PROFILING.md's clocks line), started
        # before the timed region -- its NVML start-up is over before the first timed step
        import tempfile
        try:
            self._f = tempfile.TemporaryFile(mode="w+")
            if os.environ.get("BENCH_NO_CLOCKS"):      # dev knob: no sampler
                raise RuntimeError("clock sampling disabled")
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms",
                                        os.environ.get("BENCH_CLOCK_MS", "200")],
                                       stdout=self._f, stderr=subprocess.DEVNULL, text=True)
            t0 = time.time()
            while time.time() - t0 < 3.0 and os.fstat(self._f.fileno()).st_size == 0 and self._p.poll() is None:
                time.sleep(0.02)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *exc):
        if self._p is None:
            return
        time.sleep(0.05)
        self._p.terminate()
        try:
            self._p.wait(timeout=5)
        except Exception:
            self._p.kill()
        self._f.seek(0)
        for line in self._f.read().splitlines():
            if line.strip():
                self.samples.append([x.strip() for x in line.split(",")])
        self._f.close()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _workload(cfg):
    from paper_2008_13447_b200 import gen
    c = gen.CONFIGS[cfg]
    return c, gen.series_for(cfg), gen.pair_updates(c.n, c.lmin, c.lmax)


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(path))
    except Exception:
        return {}


def cpu_sample(series, c, target_s=12.0, threads=None):
    """The oracle (C restatement of the reference's exhaustive scan) on a bounded
    sample of the same workload: whole per-length profiles at evenly spaced lengths
    until ~target_s of work. Returns (updates/s, cores, description)."""
    from oracle import oracle
    threads = threads or os.cpu_count()
    lengths = list(np.linspace(c.lmin, c.lmax, 9).astype(int))
    done, t_used, upd = [], 0.0, 0
    for L in lengths:
        t0 = time.perf_counter()
        oracle.profile(series, int(L), nthreads=threads)
        t_used += time.perf_counter() - t0
        N = series.n - L + 1
        k = N - (L + 1) // 2
        upd += k * (k + 1) // 2
        done.append(int(L))
        if t_used >= target_s:
            break
    return upd / t_used, threads, (f"full exact profiles (all rows) at lengths {done} of "
                                   f"{c.lmin}..{c.lmax}, oracle/vlmp_oracle.c, {threads} threads, "
                                   f"{t_used:.1f} s")


def _config_dict(args, c, W, world, parallelism):
    """The workload description shared by both arms (the driver compares them)."""
    return {"workload": f"config {args.config}: {c.note}", "n": c.n, "lmin": c.lmin,
            "lmax": c.lmax, "k_motif": c.k_motif, "k_discord": c.k_discord, "W_updates": W,
            "parallelism": parallelism,
            "l2": "flushed before every timed step (512 MB overwrite outside the step's event span)"}


def reference_python_sample():
    """The real reference package (baseline/_ref, its own public API and stock code path) end
    to end on config 1 -- valmod + topkm_discord_discovery, p = 50.
    Returns a dict, or None when baseline/_ref is not installed."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "seriesmine")):
        return None
    import importlib
    sys.path.insert(0, ref_dir)
    try:
        sm = importlib.import_module("seriesmine")
    finally:
        sys.path.remove(ref_dir)
    from paper_2008_13447_b200 import gen
    c = gen.CONFIGS[1]
    ds = sm.ingest(gen.series_for(1))
    W1 = gen.pair_updates(c.n, c.lmin, c.lmax)
    t0 = time.perf_counter()
    sm.valmod(ds, c.lmin, c.lmax, 50, threads=os.cpu_count())
    t1 = time.perf_counter()
    sm.topkm_discord_discovery(ds, c.lmin, c.lmax, 1, 1, 50, threads=os.cpu_count())
    t2 = time.perf_counter()
    return {"value": W1 / (t2 - t0), "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
            "sample": f"seriesmine (baseline/_ref) on config 1 (n=4096, l 32..64): valmod p=50 "
                      f"{t1 - t0:.2f} s + topkm_discord_discovery(k=1, m=1, p=50) {t2 - t1:.2f} s, "
                      f"threads={os.cpu_count()}; value = W(config 1) / total"}


def run_reference(args):
    rank, world, local = _dist_env()
    if rank != 0:
        return
    from paper_2008_13447_b200 import ingest
    c, t, W = _workload(args.config)
    s = ingest(t)
    for _ in range(args.warmup):
        cpu_sample(s, c, target_s=1.0)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, cores, desc = cpu_sample(s, c, target_s=10.0)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = float(np.mean(vals))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": _config_dict(args, c, W, world, f"{args.shard[:-1]} shards x{world}"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": desc + " (the reference's own engine cannot finish config 2 in a "
                                          "bench step: 4,863 s for valmod alone, tests/golden/make_golden.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    rank, world, local = _dist_env()
    import torch
    from paper_2008_13447_b200 import _lib, distributed, ingest
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    c, t, W = _workload(args.config)
    s = ingest(t)
    # one process per GPU; VLMP_DIST_BACKEND=gloo (host-mediated, a code-path check only)
    # lets several ranks share a device when fewer GPUs than ranks are visible
    backend = os.environ.get("VLMP_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    sess = _lib.session(local)
    k2 = max(2 * c.k_motif, 2)
    kd = max(c.k_discord, 1)

    shard_fn = distributed.profile_length_sharded if args.shard == "lengths" else distributed.profile_sharded
    parallelism = f"{args.shard[:-1]} shards x{world}"

    def step(end_event=-1):
        """One pass; with end_event the step's closing CUDA event is recorded on the stream
        behind the last read-off copy, before the host waits (one device round trip: the
        host's wake-up after it is not part of the step)."""
        if world > 1:
            shard_fn(sess, s, c.lmin, c.lmax, rank, world, group, upload=False)
            with sess.lock:
                rows = sess.smallest_rows(k2)
                disc = sess.discords(kd)
                if end_event >= 0:
                    sess.event_record(end_event)
            return rows, disc
        with sess.lock:
            sess.profile(c.lmin, c.lmax, 0, -1, 0)
            rows, disc, _ = sess.finalize_collect(k2, kd, False, end_event)
        return rows, disc

    with sess.lock:
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)   # inputs resident in HBM
    # L2 (126 MB) is flushed before every timed step by overwriting a 512 MB buffer, outside the
    # step's own CUDA-event span: each step starts cold, like the first pass over a new series
    flush_mb = int(os.environ.get("BENCH_FLUSH_MB", "512"))   # dev knob: 0 disables the flush
    flush = torch.empty(max(flush_mb, 1) << 20, dtype=torch.uint8, device="cuda")

    def flush_l2():
        if flush_mb:
            flush.zero_()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        flush_l2()
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    walk_ms, runs_ms, walk_launches, launches, step_ms_list = 0.0, 0.0, 0, 0, []
    ms = 0.0
    # one clock sampler spans both timed regions (device-resident steps, then e2e): its start-up
    # and teardown stay outside them
    clk = ClockSampler(local).__enter__()
    for _ in range(args.steps):
        flush_l2()
        sess.event_record(0)          # CUDA events on the session's stream, around the step
        rows, disc = step(end_event=1)
        one = sess.event_elapsed_ms()
        ms += one
        st = sess.stats()
        walk_ms += st["walk_ms"]
        runs_ms += st["runs_ms"]
        walk_launches += int(st["walk_launches"])
        launches += int(st["kernel_launches"]) + 2
        step_ms_list.append(one)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms, walk_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, walk_ms = float(tt[0]), float(tt[1])
        dist.barrier()
    step_ms = ms / args.steps
    value = W / (step_ms * 1e-3)

    # e2e through the public API: host arrays in, host results out, every step
    e2e_line = None
    n0 = s.n - c.lmin + 1
    nl = c.lmax - c.lmin + 1
    readoff_check = None
    if world > 1:
        # sharded: every rank uploads the host series, runs its lengths, joins the exchange and
        # builds the read-offs; rank 0's read-offs come back to the host (max over ranks)
        import torch.distributed as dist

        def e2e_step():
            shard_fn(sess, s, c.lmin, c.lmax, rank, world, group, upload=True)
            with sess.lock:
                rows = sess.smallest_rows(k2)
                disc = sess.discords(kd)
                val = sess.valmp_arrays()
            return rows, disc, val
        for _ in range(2):
            e2e_step()
        reps = max(2, min(2 * args.steps, 10))
        e2e_t = 0.0
        for _ in range(reps):
            flush_l2()
            dist.barrier()
            t0 = time.perf_counter()
            out = e2e_step()
            e2e_t += time.perf_counter() - t0
        tt = torch.tensor([e2e_t / reps], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
        e2e_line = {"value": W / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(8 * (s.n + 2 * (s.n + 1))),
                    "d2h_bytes_per_step": int(n0 * 33 + nl * (k2 * 24 + kd * 16)),
                    "ms_per_step": e2e_s * 1e3, "api": f"distributed.{shard_fn.__name__} + session read-offs"}
        if rank == 0:
            # the sharded read-offs must equal one GPU's: rank 0 re-runs the whole range alone
            with sess.lock:
                sess.profile(c.lmin, c.lmax, 0, -1, 0)
                sess.finalize()
                rows1, disc1 = sess.smallest_rows(k2), sess.discords(kd)
                val1 = sess.valmp_arrays()
            rows_n, disc_n, val_n = out
            readoff_check = bool(all(np.array_equal(a, b) for a, b in zip(rows_n, rows1))
                                 and all(np.array_equal(a, b) for a, b in zip(disc_n, disc1))
                                 and all(np.array_equal(a, b) for a, b in zip(val_n, val1)))
    if rank == 0 and world == 1:
        from paper_2008_13447_b200 import mine
        for _ in range(2):
            mine(s, c.lmin, c.lmax, k_motif=c.k_motif, k_discord=c.k_discord)
        reps = max(2, min(4 * args.steps, 20))   # enough reps for the median to shrug off host hiccups
        e2e_list = []
        for _ in range(reps):
            flush_l2()
            t0 = time.perf_counter()
            res = mine(s, c.lmin, c.lmax, k_motif=c.k_motif, k_discord=c.k_discord)
            e2e_list.append(time.perf_counter() - t0)
        # median over the reps: one host hiccup (GC, a page-in) must not set the figure; the
        # mean and every rep are reported beside it
        e2e_s = float(np.median(e2e_list))
        e2e_line = {"value": W / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(8 * (s.n + 2 * (s.n + 1))),
                    "d2h_bytes_per_step": int(n0 * (8 * 4 + 1) + nl * (2 * c.k_motif * 24 + c.k_discord * 16)),
                    "ms_per_step": e2e_s * 1e3, "ms_mean": float(np.mean(e2e_list)) * 1e3,
                    "ms_reps": [round(x * 1e3, 3) for x in e2e_list], "stat": "median of reps",
                    "api": "paper_2008_13447_b200.mine (host numpy in, host results out)"}
    clk.__exit__(None, None, None)

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    # Roofline of the dominant kernel, k_tile32 (the FP32 bound-filter walk, ~80 % of the step):
    # algorithmic work = 3 FP32 FMA per update (2 for the diagonal covariance recurrence, 1 for the
    # bound test; SURVEY.md §8(d)'s unit, W updates per step over W_l per launch -- DESIGN.md §4),
    # achieved = W * 3 FMA * 2 flop / (k_tile32 time per step, CUDA events on the launching
    # stream), peak = the measured FP32 FMA rate of this GPU (vlmp_measure_fp32_peak).
    peak_ffma = sess.measure_fp32_peak()
    peak_dfma = sess.measure_fp64_peak()
    walk_s = walk_ms * 1e-3 / args.steps
    runs_s = runs_ms * 1e-3 / args.steps
    achieved = W * 3 * 2 / walk_s / 1e12
    peak = peak_ffma * 2 / 1e12 * world
    clk_sum = clk.summary()
    prof_traffic = None
    tr_path = os.path.join(ROOT, "profiles", "tile_traffic.json")
    if os.path.exists(tr_path):
        try:
            prof_traffic = json.load(open(tr_path)).get("bytes_per_launch")
        except Exception:
            prof_traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, cores, desc = cpu_sample(s, c, target_s=12.0)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc}
        try:
            ref_py = reference_python_sample()
        except Exception as exc:           # the reference install is optional on a box
            ref_py = {"unavailable": repr(exc)[:200]}
        if ref_py is not None:
            cpu["reference_python"] = ref_py
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(args, c, W, world, parallelism),
        "step_ms_median": float(np.median(step_ms_list)),
        "step_ms": [round(x, 3) for x in step_ms_list],
        "roofline": {"bound": "fp32_fma", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": prof_traffic,
                     "kernel": "k_tile32", "launches_per_step": walk_launches / args.steps,
                     "launch_ms": walk_ms / max(walk_launches, 1),
                     "flops_per_update": "6 = 3 FP32 FMA (2 recurrence + 1 bound test) x 2; ncu counts "
                                         "3.04 executed FMA lane-ops per update (profiles/)",
                     "peak_source": "measured: vlmp_measure_fp32_peak (FFMA, all SMs, best of 3); "
                                    "MEASURED_PEAKS.json has no FP32 figure",
                     "walk_ms_per_step": walk_s * 1e3,
                     "share_of_step": walk_s * 1e3 / step_ms,
                     "chains": int(st.get("chains") or 1),
                     "chains_note": ("the length range runs as two concurrent chains on two streams (small "
                                     "series: a length's kernels do not fill the GPU back to back); walk time = "
                                     "union of the k_tile32 spans; k_runs spans overlap the other chain's walk"
                                     if (st.get("chains") or 1) > 1 else "one chain"),
                     "k_runs": {"ms_per_step": runs_s * 1e3, "share_of_step": runs_s * 1e3 / step_ms,
                                "cells_per_step": st.get("run_cells"), "bound": "fp64 / L2 latency",
                                "fp64_frac": (st.get("run_cells") or 0) * 2 / max(runs_s, 1e-12) / peak_dfma},
                     "effective_fp64_frac": W * 4 / (step_ms * 1e-3) / (peak_dfma * world),
                     "effective_fp64_note": "W x 4 FP64 FMA-pipe instr (the exhaustive FP64 cell) per step "
                                            "time over the measured DFMA peak: the FP64 work the FP32 "
                                            "filter avoids, not a pipe utilisation"},
        "cpu_baseline": cpu,
        "e2e": e2e_line,
        "gpu_launches": launches,
        "graph": bool(st.get("graph")),
        "clocks": clk_sum,
    }
    if readoff_check is not None:
        line["readoffs_equal_1gpu"] = readoff_check
        line["dist_backend"] = backend
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = _args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    if args.gpus > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # communicator lines show the rank count
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
