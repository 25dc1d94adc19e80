#!/usr/bin/env python3
"""Benchmark: the accelerated spherical k-means loop on B200 vs the reference's CPU path.

Workload (BASELINE.json configs[3], "C4", the largest single-GPU config and
the one north_star's targets are stated on): n = 4,000,000 synthetic TF-IDF
docs, d = 1,000,000, mean ~60 nnz/row, Zipf(1.1) terms with 1,000 planted
topics (seeded, paper_2107_04074_b200/synth.py), k = 1,000, uniform seeded
init (seed 2), max_iter 50.  One STEP = one complete fit of each of
BASELINE's C4 variants (hamerly, simp_elkan) from the same start.
metric = k-means iterations/s over the step (plus effective n*k sims/s and
the pruned fraction as extra keys).  ``--config/--k/--variants`` select the
other configs (C2, C3, C5) for profiling runs.

  value      device-timed (CUDA events per step, inputs resident in HBM;
             the C4 working set is far larger than L2, and L2 is also
             flushed before every step)
  e2e        same work through the public API from pinned HOST buffers:
             every step the raw CSR rows are copied H2D into the serving
             buffers (device layout rebuilt on the GPU), seed row ids H2D,
             stats + assignments D2H
  roofline   the dominant kernel (by CUDA-event time in an instrumented
             pass) with its algorithmic bytes / time, next to every other
             kernel's; the ncu DRAM traffic per launch from profiles/
  cpu_baseline  the CPU oracle (C port of the reference loop, OpenMP) on a
             bounded sample, rank 0 at N=1 only; cpu_baseline_reference:
             the unmodified reference package (baseline/_ref, 1 core)

--impl reference runs the oracle port (C, all host threads) on a bounded
sample of the same workload: the first n' rows of the corpus, each variant
capped at a few iterations, its row-proportional phase time scaled by
n / n' (the oracle's phase clocks; the k x d center phases are not scaled).
That process never loads the product library (rows are normalised by the
oracle's np.dot-order row norms).

Multi-GPU (``--gpus N``; re-executed under torch.distributed.run when
WORLD_SIZE is unset): the corpus is replicated, every rank scans an
nnz-balanced shard of the rows, and one NCCL allgather of the packed moves
per iteration keeps the replicated int64 fixed-point sums identical on all
ranks (paper_2107_04074_b200/distributed.py); weak in memory, strong in
work (total work fixed).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

VARIANTS = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
DEFAULTS = {"C1": (20, VARIANTS), "C2": (100, VARIANTS), "C3": (200, ("elkan", "hamerly")),
            "C4": (1000, ("hamerly", "simp_elkan")), "C5": (1000, ("hamerly",))}
PEAKS = ROOT / "MEASURED_PEAKS.json"
REF_STEP_S = 5.0          # target seconds of CPU work per reference-arm step


def metric_name(args) -> str:
    """BASELINE.json's iterations/s metric, labelled with the workload."""
    return f"k-means iterations/s ({args.config}, k={args.k}, {len(args.variants.split(','))} variants per step)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--n", type=int, default=None, help="row count override (the generator at n rows)")
    p.add_argument("--seed", type=int, default=2)
    p.add_argument("--max-iter", type=int, default=50)
    p.add_argument("--variants", default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (A/B runs)")
    p.add_argument("--no-roofline", action="store_true", help="skip the instrumented pass (A/B runs)")
    p.add_argument("--profile-only", action="store_true", help="one untimed step (for ncu)")
    a = p.parse_args()
    k0, v0 = DEFAULTS.get(a.config, (100, VARIANTS))
    a.k = a.k if a.k is not None else k0
    a.variants = a.variants if a.variants is not None else ",".join(v0)
    if a.warmup < 1:
        a.warmup = 1
    return a


def maybe_launch_ranks(args) -> bool:
    """--gpus N > 1 outside torchrun: re-execute this command under
    torch.distributed.run with N ranks (one per GPU).  Returns True if it did."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    rc = subprocess.call(cmd)
    sys.exit(rc)


def peaks():
    try:
        return json.loads(PEAKS.read_text()), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


class Clocks:
    """NVML sampler (every 5 ms) running during the timed region: SM clock + throttle reasons."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0, period=0.005):
        self.index, self.period = index, period
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report why
            self.error = repr(e)
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((float(sm), int(rs)))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(1.0)
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "note": getattr(self, "error", "no samples")}
        sm = [s for s, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "nvml every 5 ms"}


# ----------------------------------------------------------------- workload
def load_workload(args, host_only: bool = False):
    """The config's Dataset.  host_only (reference arm): rows normalised with
    the oracle's np.dot-order row norms, so the product library is never loaded."""
    from paper_2107_04074_b200 import synth
    norms = None
    if host_only:
        from oracle import oracle as O
        norms = O.row_norms
    t = time.time()
    data = synth.config_dataset(args.config, n_override=args.n, row_norms=norms)
    return data, time.time() - t


def workload_config(args, data, n_gpus):
    return {"workload": f"{args.config} n={data.n} d={data.dim} nnz={data.nnz} k={args.k}; "
                        f"one step = one fit of each of [{args.variants}] (seed {args.seed}, max_iter {args.max_iter})",
            "global_batch": data.n, "k": args.k, "variants": args.variants.split(","),
            "parallelism": (f"dp{n_gpus} (corpus replicated, rows sharded by nnz, centers replicated, "
                            f"one allgather of moves per iteration)" if n_gpus > 1 else "single GPU"),
            "l2": "flushed (256 MiB write) before every timed step; C4's working set (CSR 2 GB, center table "
                  "4 GB) is also far larger than L2",
            "precision": "fp32 similarities, fp64 centers, exact int64 fixed-point sums"}


# ----------------------------------------------------------------- CPU legs
D_FOLD = 20000     # columns of the CPU samples: the k x d center phases scale linearly in d


def cpu_sample(data, n_sub: int, d_fold: int = D_FOLD):
    """The CPU legs' sample: the first n_sub rows; when d > d_fold, term ids
    folded modulo d_fold (duplicates within a row summed, rows renormalised),
    so the k x d center phases (thresholds, renormalise, objective: linear in
    d) cost d_fold/d of the full size and are scaled back by d/d_fold.  The
    row phases keep every nnz (their cost does not depend on d, except that a
    smaller center table caches better on the host: conservative for the GPU).
    Returns (indptr, int32 indices, float64 data, d_sample)."""
    n_sub = min(n_sub, data.n)
    ip = np.asarray(data.indptr[:n_sub + 1], np.int64)
    ix = np.asarray(data.indices[:ip[-1]], np.int64)
    dv = np.asarray(data.data[:ip[-1]], np.float64)
    if data.dim <= d_fold:
        return ip, ix.astype(np.int32), dv, data.dim
    rows = np.repeat(np.arange(n_sub, dtype=np.int64), np.diff(ip))
    key = rows * d_fold + ix % d_fold
    order = np.argsort(key, kind="stable")
    ks = key[order]
    uniq, start = np.unique(ks, return_index=True)
    vals = np.add.reduceat(dv[order], start)
    keep = vals != 0.0
    uniq, vals = uniq[keep], vals[keep]
    r = uniq // d_fold
    counts = np.bincount(r, minlength=n_sub)
    if np.any(counts == 0):
        raise ValueError("a folded sample row is empty")
    ip2 = np.zeros(n_sub + 1, np.int64)
    np.cumsum(counts, out=ip2[1:])
    nrm = np.sqrt(np.add.reduceat(vals * vals, ip2[:-1]))
    vals = vals / np.repeat(nrm, counts)
    return ip2, (uniq % d_fold).astype(np.int32), vals, d_fold


def _oracle_sample(data, n_sub: int):
    """(oracle CSR of the CPU sample, d / d_sample)."""
    from oracle import oracle as O
    ip, ix, dv, ds = cpu_sample(data, n_sub)
    return O.CSR(ip, ix, dv, ds), data.dim / ds


def oracle_plan(args, data, budget_s: float):
    """(n_sub, max_iter) so that one fit of every variant on the first n_sub
    rows costs about budget_s of CPU time: a 2-iteration probe on at most 20k
    rows measures the row-proportional and the center (k x d) phase costs."""
    from oracle import oracle as O
    variants = args.variants.split(",")
    k = args.k
    n_probe = min(data.n, max(5000, 4 * k))
    X, dscale = _oracle_sample(data, n_probe)
    r = O.run(X, min(k, n_probe), variants[0], seed=args.seed, max_iter=2)
    its = max(r["iterations"], 1)
    per_row = float(r["t_rows"].sum()) / its / n_probe
    other = float(r["t_other"].sum()) / its          # at the sample's d: the measured share of a step
    mi = min(args.max_iter, 50)
    per_it_full = per_row * data.n + other
    if per_it_full * mi * len(variants) <= budget_s:
        return data.n, mi
    mi = max(2, min(mi, 4))
    room = budget_s / (mi * len(variants)) - other
    n_sub = int(room / per_row) if room > 0 else n_probe
    n_sub = max(min(data.n, max(2 * k, 5000)), min(data.n, n_sub))
    return n_sub, mi


def oracle_sample_rate(args, data, n_sub: int, mi: int):
    """One fit of every variant on the first n_sub rows (cap mi iterations):
    (iterations, full-size-equivalent seconds, measured seconds)."""
    from oracle import oracle as O
    X, dscale = _oracle_sample(data, n_sub)
    its, t_full, t_meas = 0, 0.0, 0.0
    for v in args.variants.split(","):
        r = O.run(X, min(args.k, n_sub), v, seed=args.seed, max_iter=mi)
        its += r["iterations"]
        tr, to = float(r["t_rows"].sum()), float(r["t_other"].sum())
        t_meas += tr + to
        t_full += tr * data.n / n_sub + to * dscale
    return its, t_full, t_meas


def sample_label(data, n_sub, mi, args):
    if n_sub >= data.n and mi >= args.max_iter:
        return f"full workload: one fit of each of [{args.variants}]"
    rows = "all rows" if n_sub >= data.n else f"the first {n_sub} of {data.n} rows"
    fold = (f", term ids folded to d' = {D_FOLD} (k x d center phases -- thresholds, renormalise, objective -- "
            f"timed at d' and scaled by d/d' = {data.dim / D_FOLD:g})" if data.dim > D_FOLD else
            ", k x d center phases counted as measured")
    return (f"one fit of each of [{args.variants}] on {rows}, each capped at {mi} iterations; "
            f"row-proportional phase time (sims, bounds, scans, aggregation, moves) scaled by n/n_sub" + fold)


def run_reference(args):
    """--impl reference: the oracle port on the box's host cores, bounded sample per step."""
    from oracle import oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    data, _ = load_workload(args, host_only=True)
    cores = O.num_threads()
    n_sub, mi = oracle_plan(args, data, REF_STEP_S)
    for _ in range(args.warmup):
        oracle_sample_rate(args, data, n_sub, mi)
    its_tot, tf_tot, tm_tot = 0, 0.0, 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        its, tf, tm = oracle_sample_rate(args, data, n_sub, mi)
        its_tot, tf_tot, tm_tot = its_tot + its, tf_tot + tf, tm_tot + tm
    wall = time.perf_counter() - t0
    val = its_tot / tf_tot
    sample = sample_label(data, n_sub, mi, args) + f"; {args.steps} steps, {wall:.1f} s measured wall"
    line = {"metric": metric_name(args), "value": val, "unit": "iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tf_tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload_config(args, data, 1),
                                                precision="float64 (C port of the reference loop, the oracle)"),
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, data, budget_s: float = 20.0):
    """The oracle port on a bounded sample (about budget_s of CPU work)."""
    from oracle import oracle as O
    n_sub, mi = oracle_plan(args, data, budget_s)
    its, tf, tm = oracle_sample_rate(args, data, n_sub, mi)
    return {"value": its / tf, "unit": "iterations/s", "cores": O.num_threads(), "kind": "port",
            "sample": sample_label(data, n_sub, mi, args) + f" ({its} iterations, {tm:.1f} s measured)"}


def cpu_baseline_reference(args, data, n_sub: int = 10000, max_iter: int = 3, timeout: int = 900):
    """The unmodified reference package (baseline/_ref) on 1 core, first n_sub rows,
    max_iter iterations per variant (baseline/ref_sample.py, own process)."""
    if not (ROOT / "baseline" / "_ref" / "spkmeans").exists():
        return {"unavailable": "baseline/_ref not installed"}
    n_sub = min(n_sub, data.n)
    ip, ix, dv, ds = cpu_sample(data, n_sub)
    with tempfile.TemporaryDirectory() as td:
        f = Path(td) / "sample.npz"
        np.savez(f, indptr=ip, indices=ix, data=dv, dim=ds)
        cmd = [sys.executable, str(ROOT / "baseline" / "ref_sample.py"), "--npz", str(f), "--k",
               str(min(args.k, n_sub)), "--variants", args.variants, "--max-iter", str(max_iter), "--seed",
               str(args.seed), "--n-full", str(data.n), "--d-full", str(data.dim)]
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
            r = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception as e:
            return {"unavailable": f"reference sample failed: {e!r}"[:300]}
    if "unavailable" in r:
        return r
    return {"value": r["its_per_s_full_est"], "unit": "iterations/s", "cores": 1, "kind": "reference",
            "sample": (f"unmodified spkmeans {r['spkmeans']} (baseline/_ref), serial: one fit of each of "
                       f"[{args.variants}] on the first {r['n_sub']} of {data.n} rows, max_iter {max_iter}; "
                       f"row phases scaled by n/n_sub, k x d center phases "
                       + (f"timed at folded d' = {ds} and scaled by d/d'" if ds < data.dim else "as measured")),
            "value_at_sample": r["its_per_s_sample"], "detail": r}


# ----------------------------------------------------------------- our arm
def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import _lib
    from paper_2107_04074_b200.engine import DeviceCorpus, run
    from paper_2107_04074_b200.seeding import SeedConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    data, gen_s = load_workload(args)
    variants = args.variants.split(",")
    k = args.k
    if world > 1:
        from paper_2107_04074_b200.distributed import Exchange
    rows = (0, data.n)                 # multi-GPU: corpus replicated, scans sharded (distributed.py)
    corpus = DeviceCorpus(data, dev, rows=rows)
    torch.cuda.synchronize()

    exchanges = {}     # one Exchange per corpus (multi-GPU): engines are cached per (corpus, exchange)

    def exchange_for(corpus_):
        if id(corpus_) not in exchanges:
            exchanges[id(corpus_)] = Exchange.for_corpus(k, corpus_, dev)
        return exchanges[id(corpus_)]

    def fit_all(corpus_):
        its, sims, nk = 0, 0, 0
        per = {}
        for v in variants:
            comm = exchange_for(corpus_) if world > 1 else None
            r = run(data, k, v, SeedConfig(seed=args.seed), max_iter=args.max_iter, device=dev, corpus=corpus_,
                    comm=comm, n_total=data.n)
            its += len(r.iterations)
            sims += r.total_sims
            nk += data.n * k * len(r.iterations)
            per[v] = {"iterations": len(r.iterations), "objective": r.objective,
                      "pruned_frac": 1.0 - r.total_sims / (data.n * k * len(r.iterations))}
        return its, sims, nk, per

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if args.profile_only:
        fit_all(corpus)
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        fit_all(corpus)
    # ---- device-timed steps (inputs resident) ----
    times, its_tot, sims_tot, nk_tot = [], 0, 0, 0
    prof = _lib.CallProfiler(timed=False)
    gc.collect()
    gc.disable()                      # no collector pauses between the fits of a timed step
    with Clocks(local) as clk:
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            with prof:
                its, sims, nk, per = fit_all(corpus)
            e1.record()
            barrier()
            times.append(e0.elapsed_time(e1))
            its_tot, sims_tot, nk_tot = its_tot + its, sims_tot + sims, nk_tot + nk
    gc.enable()
    step_ms = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(step_ms, op=dist.ReduceOp.MAX)
    total_ms = float(step_ms.item())
    value = its_tot / (total_ms / 1e3)
    launches_per_step = prof.launches // max(args.steps, 1)

    # ---- e2e through the public API from host buffers ----
    # every step: the CSR's host arrays (page-locked in place) are uploaded
    # (raw rows H2D; device-order layout, term renumbering and float32
    # conversion rebuilt on the GPU) into the serving buffers of a persistent
    # DeviceCorpus, then the user's call spk.run(...) per variant (seed row
    # ids H2D, stats + assignments D2H).  Untimed warm-up steps fill the
    # engine cache for that corpus and capture its fit graphs.
    e2e = None
    if not args.no_e2e:
        e2e_times, h2d, d2h = [], 0, 0
        del corpus
        from paper_2107_04074_b200 import engine as _E
        _E.clear_engine_cache()
        torch.cuda.empty_cache()
        c = DeviceCorpus(data, dev, rows=rows, pinned_host=True)

        def e2e_step():
            c.refresh(data)
            b_in, b_out = c.h2d_bytes, 0
            for v in variants:
                comm = exchange_for(c) if world > 1 else None
                r = spk.run(data, k, v, SeedConfig(seed=args.seed), max_iter=args.max_iter, device=dev, corpus=c,
                            comm=comm, n_total=data.n)
                b_in += int(k * 8)
                b_out += r.assignments.nbytes + 8 * len(r.iterations) * _lib.ST_COUNT
            return b_in, b_out

        for _ in range(max(args.warmup, 2)):
            e2e_step()
        barrier()
        gc.collect()
        gc.disable()
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h2d, d2h = e2e_step()
            e1.record()
            barrier()
            e2e_times.append(e0.elapsed_time(e1))
        gc.enable()
        e2e_ms = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": its_tot / (float(e2e_ms.item()) / 1e3), "unit": "iterations/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
        corpus = c

    # ---- instrumented pass: per-entry-point event times -> roofline ----
    roof = None if args.no_roofline else roofline(args, data, corpus, dev, world)

    if rank != 0:
        dist.destroy_process_group()
        return
    clocks = clk.summary()
    line = {"metric": metric_name(args), "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, data, world),
            "effective_sims_per_s": nk_tot / (total_ms / 1e3),
            "computed_sims_per_s": sims_tot / (total_ms / 1e3),
            "pruned_frac": 1.0 - sims_tot / nk_tot,
            "per_variant": per,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof,
            "clocks": clocks,
            "data_gen_s": round(gen_s, 1)}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, data)
        line["cpu_baseline_reference"] = cpu_baseline_reference(args, data)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# entry point -> the kernel doing its work (the dominant kernel is chosen
# per KERNEL, so entry points sharing one kernel are pooled)
KERNEL_OF = {"spkm_full_assign": "k_row_pass", "spkm_hamerly_rescan": "k_row_pass",
             "spkm_hamerly_tighten": "k_hamerly_tighten", "spkm_hamerly_bounds": "k_hamerly_bounds",
             "spkm_elkan_bounds": "k_elkan_bounds", "spkm_elkan_scan": "k_elkan_scan / k_elkan_light",
             "spkm_elkan_heavy": "k_row_pass",
             "spkm_elkan_bounds_scan": "k_elkan_scan (fused bounds)", "spkm_dense_assign": "k_dense_pass",
             "spkm_apply_moves": "k_apply_moves", "spkm_aggregate_sums": "k_aggregate",
             "spkm_order_by_cluster": "k_order_*", "spkm_move_centers": "center pipeline (4 kernels)",
             "spkm_center_thresholds": "k_gram_mn + k_gram_final + k_row_max",
             "spkm_yy_bounds": "k_yy_bounds", "spkm_yy_scan": "k_yy_scan"}
MULTI = {"spkm_move_centers", "spkm_center_thresholds", "spkm_order_by_cluster"}


def roofline(args, data, corpus, dev, world):
    """Time every entry point with CUDA events (on the stream its kernels run
    on) over one eager step; algorithmic bytes per SURVEY.md §8(d) from the
    fits' own counters; aggregate per kernel."""
    import torch
    from paper_2107_04074_b200 import _lib
    from paper_2107_04074_b200.engine import run
    from paper_2107_04074_b200.distributed import Exchange
    from paper_2107_04074_b200.seeding import SeedConfig

    pk, src = peaks()
    n, nnz, k = corpus.n, corpus.nnz, args.k
    dense = getattr(corpus, "dense_dim", None) is not None
    prof = _lib.CallProfiler(timed=True)
    bytes_by, flops_by, gather_by = {}, {}, {}
    kp = int(_lib.lib().spkm_padded_k(k))
    ku = (k + 3) // 4 * 4
    with prof:
        for v in args.variants.split(","):
            prof.tag = v
            comm = Exchange.for_corpus(k, corpus, dev) if world > 1 else None
            r = run(data, k, v, SeedConfig(seed=args.seed), max_iter=args.max_iter, device=dev, corpus=corpus,
                    comm=comm, n_total=data.n)
            its = r.iterations
            csr_row = 12          # int64 indptr + fp32 row eps per row read
            csr_full = 8 * nnz + csr_row * n
            n_full = 1 + (len(its) - 1 if v == "standard" else 0)
            # full passes: CSR + the bound writes (a, l; u: Hamerly 4 B, Elkan 4k B)
            gpw = ((k + 3) // 4 + 3) // 4 * 4
            init_w = 8 * n + (4 * ku * n if v in ("elkan", "simp_elkan") else 4 * n if "hamerly" in v
                              else 4 * gpw * n if v == "yinyang" else 0)
            b = csr_full * n_full + init_w + 4 * n * (n_full - 1)
            bytes_by[("spkm_full_assign", v)] = b
            gather_by[("spkm_full_assign", v)] = 4 * kp * nnz * n_full
            if v in ("hamerly", "simp_hamerly"):
                # bound pass: a, l, u, eps read; l, u written; survivor ids written
                bytes_by[("spkm_hamerly_bounds", v)] = sum(24 * n + 4 * s.survivors for s in its[1:])
                # tighten + rescan: both pooled under k_row_pass/k_hamerly_tighten by time; the bytes of
                # the tighten test (CSR of the bound survivors) are credited to whichever ran it
                tb = sum(8 * s.nnz_tighten + (csr_row + 12) * s.survivors for s in its[1:])
                rb = sum(8 * s.nnz_rescan + (csr_row + 12) * s.survivors2 for s in its[1:])
                bytes_by[("spkm_hamerly_scan", v)] = tb + rb
                gather_by[("spkm_hamerly_scan", v)] = sum(4 * kp * s.nnz_rescan + 4 * s.nnz_tighten for s in its[1:])
            if v in ("elkan", "simp_elkan"):
                # bound pass: u read (4 ku) + a, l, eps (12) + l write (4) per row, and u written only in
                # the 16-byte groups holding a center that moved (touched clusters of the previous iteration)
                moved_prev = [its[q - 1].touched for q in range(1, len(its))]
                # the bound pass is skipped (every row takes the full pass) in an iteration that follows one
                # which moved >= n / 256 rows (spkm_work.allheavy_rows; only with the heavy-row pass, k > 256)
                heavy_on = any(s.survivors2 for s in its[1:]) and os.environ.get("SPKM_EK_ALLHEAVY", "1") != "0"
                ran = [not (heavy_on and 256 * its[q - 1].reassignments >= n) for q in range(1, len(its))]
                b_bounds = sum(((4 * ku + 16) * n + 4 * min(ku, 4 * m) * n) for m, r_ in zip(moved_prev, ran) if r_)
                # light rows scanned from the bound pass's lists (k_elkan_light: simp_elkan, heavy threshold <= 5):
                # the 16-byte list, a / l / eps, and the <= 5 u(i, j) touched instead of the whole u row
                lists = (v == "simp_elkan" and any(s.survivors2 for s in its[1:]) and (k + 199) // 200 <= 5
                         and os.environ.get("SPKM_EK_LIGHT", "1") != "0" and not os.environ.get("SPKM_EK_HEAVY_PCT"))
                per_surv = (csr_row + 16 + 16 + 40) if lists else (csr_row + 4 * ku + 16)
                b_scan = sum(8 * s.nnz_elkan + per_surv * s.survivors for s in its[1:])
                bytes_by[("spkm_elkan_bounds", v)] = b_bounds
                bytes_by[("spkm_elkan_scan", v)] = b_scan
                # heavy rows (spkm_elkan_heavy, k > 256): CSR row + a, l, eps, and every u(i, j) written
                b_heavy = sum(8 * s.nnz_rescan + (csr_row + 4 * ku + 12) * s.survivors2 for s in its[1:])
                if b_heavy:
                    bytes_by[("spkm_elkan_heavy", v)] = b_heavy
                    gather_by[("spkm_elkan_heavy", v)] = sum(4 * kp * s.nnz_rescan for s in its[1:])
                # fused: the scan's u reads of a survivor are the bound pass's (counted once)
                bytes_by[("spkm_elkan_bounds_scan", v)] = b_bounds + sum(
                    8 * s.nnz_elkan + csr_row * s.survivors for s in its[1:])
            if v == "yinyang":
                # group bounds (4 centers per group, gp per row): bound pass reads ug, a, l, eps, writes l and
                # the groups holding a moved center; the scan re-reads the survivor's CSR row and ug
                gp = ((k + 3) // 4 + 3) // 4 * 4
                moved_prev = [its[q - 1].touched for q in range(1, len(its))]
                bytes_by[("spkm_yy_bounds", v)] = sum((4 * gp + 16) * n + 4 * min(gp, m) * n for m in moved_prev)
                bytes_by[("spkm_yy_scan", v)] = sum(8 * s.nnz_elkan + (csr_row + 8 * gp + 16) * s.survivors
                                                    for s in its[1:])
            bytes_by[("spkm_apply_moves", v)] = sum(16 * s.nnz_moved for s in its[1:])
            bytes_by[("spkm_move_centers", v)] = sum(20 * s.touched * data.dim for s in its)
            if dense:
                D = corpus.dense_dim
                rows = n * n_full + (sum(s.survivors for s in its[1:]) if "hamerly" in v else 0)
                flops_by[("spkm_dense_assign", v)] = 2 * rows * k * D     # the algorithm's flops (k, not kpad)
    torch.cuda.synchronize()
    times = prof.times_ms()
    calls = {}
    for (name, tag), ms in times.items():
        key = "spkm_hamerly_scan" if name in ("spkm_hamerly_tighten", "spkm_hamerly_rescan") else name
        calls.setdefault(key, [0.0, 0])
        calls[key][0] += ms
    for name, e0, e1, tag in prof.records:
        key = "spkm_hamerly_scan" if name in ("spkm_hamerly_tighten", "spkm_hamerly_rescan") else name
        calls[key][1] += 1
    total = sum(v[0] for v in calls.values())
    share = {nm: round(v[0] / total, 4) for nm, v in sorted(calls.items(), key=lambda x: -x[1][0])}

    def entry_bytes(nm):
        return sum(val for key, val in bytes_by.items() if key[0] == nm)

    per = {}
    for nm, (ms, nl) in calls.items():
        b = entry_bytes(nm)
        if b and ms:
            per[nm] = {"kernel": KERNEL_OF.get(nm, "k_row_pass (rescan) + k_hamerly_tighten"), "launches": nl,
                       "ms": round(ms, 4), "algorithmic_bytes": b,
                       "achieved_gbs": round(b / (ms / 1e3) / 1e9, 1),
                       "frac": round(b / (ms / 1e3) / 1e9 / pk.get("hbm_gbs"), 4)}
    out = {"bound": "hbm", "peak": pk.get("hbm_gbs"), "unit": "GB/s", "peak_source": src + ", copy bandwidth",
           "time_share": share, "traffic": None}
    cand = [nm for nm in share if nm not in MULTI and (entry_bytes(nm) or any(key[0] == nm for key in flops_by))]
    # the dominant KERNEL: entry points that run the same kernel are pooled (k_row_pass serves the
    # full passes, the Hamerly rescan -- its tighten launch is a no-op when fused -- and the Elkan heavy rows)
    def kernel_of(nm):
        return "k_row_pass" if nm == "spkm_hamerly_scan" else KERNEL_OF.get(nm, nm)
    groups = {}
    for nm in cand:
        groups.setdefault(kernel_of(nm), []).append(nm)
    dom_group = max(groups.values(), key=lambda g: sum(calls[x][0] for x in g)) if groups else []
    dom = dom_group[0] if dom_group else None      # its largest entry point (share is sorted by time)
    if dom and any(key[0] == dom for key in flops_by):
        ms = calls[dom][0]
        f = sum(val for key, val in flops_by.items() if key[0] == dom)
        peak_tf32, how = tf32_peak(dev)
        ach = f / (ms / 1e3) / 1e12
        out.update({"bound": "tensor", "unit": "TFLOP/s", "kernel": KERNEL_OF[dom], "entry": dom, "achieved": ach,
                    "peak": peak_tf32, "peak_source": how, "frac": ach / peak_tf32, "launches": calls[dom][1],
                    "algorithmic_flops": f, "kernel_ms": ms,
                    "note": "2 n k D flops per pass over the kernel's CUDA-event time (3xTF32 issues 3 MMAs each)"})
    elif dom:
        ms = sum(calls[x][0] for x in dom_group)
        b = sum(entry_bytes(x) for x in dom_group)
        ach = b / (ms / 1e3) / 1e9
        out.update({"kernel": kernel_of(dom), "entry": dom, "entries": dom_group, "achieved": ach,
                    "frac": ach / pk.get("hbm_gbs"), "launches": sum(calls[x][1] for x in dom_group),
                    "algorithmic_bytes": b, "kernel_ms": ms})
    tr = ncu_traffic(args.config, dom)
    if tr is not None:
        out["traffic"] = tr.get("dram_bytes_per_launch")
        out["traffic_source"] = tr.get("source")
        for key in ("algorithmic_bytes_per_launch", "ncu_throughput_pct", "note"):
            if key in tr:
                out["traffic_" + key] = tr[key]
    out["per_kernel"] = per
    # the whole step on SURVEY 8(d)'s definition: B_iter = CSR bytes + bound bytes of every pass (center
    # update and move bytes are reported separately, below), over the instrumented step's kernel time
    iter_entries = [nm for nm in calls if nm not in ("spkm_move_centers", "spkm_apply_moves") and entry_bytes(nm)]
    b_iter = sum(entry_bytes(nm) for nm in iter_entries)
    if b_iter and total:
        out["step"] = {"algorithmic_bytes": b_iter, "ms": round(total, 3),
                       "achieved_gbs": round(b_iter / (total / 1e3) / 1e9, 1),
                       "frac": round(b_iter / (total / 1e3) / 1e9 / pk.get("hbm_gbs"), 4),
                       "note": "sum of CSR + bound bytes of all passes / sum of all kernels' event time of one step"}
    # the gather passes are bound by the center-row gathers (L2/DRAM), not by
    # their CSR bytes: the center-row bytes they pull per second
    gv = {}
    for nm, (ms, nl) in calls.items():
        g = sum(val for key, val in gather_by.items() if key[0] == nm)
        if g and ms:
            gv[nm] = {"center_row_bytes": g, "ms": round(ms, 4), "achieved_gbs": round(g / (ms / 1e3) / 1e9, 1)}
    if gv:
        out["center_gather"] = gv
    if "spkm_move_centers" in calls:
        b = entry_bytes("spkm_move_centers")
        ms = calls["spkm_move_centers"][0]
        out["center_update"] = {"entry": "spkm_move_centers", "algorithmic_bytes": b, "ms": ms,
                                "achieved_gbs": b / (ms / 1e3) / 1e9 if ms else None,
                                "note": "20 B per (touched cluster, term), SURVEY.md 8(d); event span of 4 kernels"}
    return out


def tf32_peak(dev):
    """Measured dense TF32 tensor throughput (cuBLAS via torch, 8192^3, best of 5)."""
    import torch
    try:
        old = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(8192, 8192, device=dev)
        b = torch.randn(8192, 8192, device=dev)
        best = 0.0
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        torch.backends.cuda.matmul.allow_tf32 = old
        return best, "measured: cuBLAS TF32 GEMM 8192^3 in bench.py"
    except Exception as e:  # pragma: no cover
        return 1100.0, f"nominal dense TF32 ({e!r})"


def ncu_traffic(config, entry):
    """DRAM bytes per launch of the entry's kernel from a committed ncu --set full capture of this config."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if entry is None or not p.exists():
        return None
    try:
        t = json.loads(p.read_text())
        return t.get(config, {}).get(entry)
    except Exception:
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    maybe_launch_ranks(args)
    main_ours(args)


if __name__ == "__main__":
    main()
