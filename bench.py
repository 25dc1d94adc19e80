#!/usr/bin/env python3
"""Benchmark: the accelerated spherical k-means loop on B200 vs the reference's CPU path.

Workload (BASELINE.json configs[1], "C2"): n=20,000 synthetic TF-IDF docs,
d=100,000, mean ~120 nnz/row (Zipf(1.1) terms, lognormal lengths; seeded,
see paper_2107_04074_b200/synth.py), k=100, uniform seeded init (seed 2),
max_iter 50.  One STEP = one complete fit of each of the five variants
(standard, elkan, simp_elkan, hamerly, simp_hamerly) from the same start.
metric = k-means iterations/s over the step (plus effective n*k sims/s and
the pruned fraction as extra keys).

  value      device-timed (CUDA events per step, inputs resident in HBM)
  e2e        same work through the public API from pinned HOST buffers:
             every step the raw CSR rows are copied H2D into the serving
             buffers (device layout rebuilt on the GPU), seed row ids H2D,
             stats + assignments D2H
  roofline   the dominant kernel's algorithmic bytes / its event time
  cpu_baseline  the CPU oracle (C port of the reference loop, OpenMP over
             points) on a bounded sample, rank 0 at N=1 only

--impl reference runs the oracle port (the reference package is Python and
cannot travel to the GPU box) on the same workload.  Multi-GPU (torchrun):
rows sharded by nnz, one allreduce per iteration; strong scaling.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

VARIANTS = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
def metric_name(args) -> str:
    """BASELINE.json's iterations/s metric, labelled with the workload (C2, k=100, 5 variants by default)."""
    return f"k-means iterations/s ({args.config}, k={args.k}, {len(args.variants.split(','))} variants per step)"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2")
    p.add_argument("--k", type=int, default=100)
    p.add_argument("--n", type=int, default=None, help="row count override (subsample of the config)")
    p.add_argument("--seed", type=int, default=2)
    p.add_argument("--max-iter", type=int, default=50)
    p.add_argument("--variants", default=",".join(VARIANTS))
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-only", action="store_true", help="one untimed step (for ncu)")
    return p.parse_args()


def peaks():
    try:
        return json.loads(PEAKS.read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


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
def load_workload(args):
    from paper_2107_04074_b200 import synth
    t = time.time()
    data = synth.config_dataset(args.config, n_override=args.n)
    return data, time.time() - t


def workload_config(args, data, n_gpus):
    return {"workload": f"{args.config} n={data.n} d={data.dim} nnz={data.nnz} k={args.k}; "
                        f"one step = one fit of each of [{args.variants}] (seed {args.seed}, max_iter {args.max_iter})",
            "global_batch": data.n, "k": args.k, "variants": args.variants.split(","),
            "parallelism": f"dp{n_gpus} (rows sharded by nnz, centers replicated)",
            "l2": "flushed (256 MiB write) before every timed step",
            "precision": "fp32 similarities, fp64 centers, exact int64 fixed-point sums"}


# ----------------------------------------------------------------- reference arm
def run_reference(args):
    from oracle import oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    data, _ = load_workload(args)
    X = O.CSR(data.indptr, data.indices, data.data, data.dim)
    variants = args.variants.split(",")
    cores = O.num_threads()

    def step():
        its = 0
        for v in variants:
            r = O.run(X, args.k, v, seed=args.seed, max_iter=args.max_iter)
            its += r["iterations"]
        return its

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    its = sum(step() for _ in range(args.steps))
    dt = time.perf_counter() - t0
    val = its / dt
    line = {"metric": metric_name(args), "value": val, "unit": "iterations/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args, data, args.gpus),
                           precision="float64 (C port of the reference loop, the oracle)"), "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": cores, "kind": "port",
                             "sample": f"full workload ({args.steps} steps x {len(variants)} fits), OpenMP over points"},
            "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, data, budget_s: float = 20.0):
    """Bounded sample (about 10-30 s of CPU): one fit of each variant with the
    oracle.  A 2-iteration probe on at most 20k rows estimates the cost; when
    the full workload does not fit the budget the fits are capped in
    iterations and, if needed, run on the first n' rows with the rate scaled
    by n'/n (per-iteration cost is linear in n), and the sample says so."""
    from oracle import oracle as O
    variants = args.variants.split(",")

    def csr(rows):
        ip = data.indptr[:rows + 1]
        return O.CSR(ip, data.indices[:ip[-1]], data.data[:ip[-1]], data.dim)

    n_probe = min(data.n, 20000)
    t0 = time.perf_counter()
    probe = O.run(csr(n_probe), min(args.k, n_probe), variants[0], seed=args.seed, max_iter=2)["iterations"]
    per_it_full = (time.perf_counter() - t0) / max(probe, 1) * data.n / n_probe
    n_sub, mi = data.n, args.max_iter
    if per_it_full * mi * len(variants) > budget_s:
        mi = max(2, min(mi, int(budget_s / (per_it_full * len(variants)))))
        if per_it_full * mi * len(variants) > budget_s:
            n_sub = max(min(data.n, 2000), int(data.n * budget_s / (per_it_full * mi * len(variants))))
    X = csr(n_sub) if n_sub < data.n else O.CSR(data.indptr, data.indices, data.data, data.dim)
    its = 0
    t0 = time.perf_counter()
    for v in variants:
        its += O.run(X, min(args.k, n_sub), v, seed=args.seed, max_iter=mi)["iterations"]
    dt = time.perf_counter() - t0
    scale = n_sub / data.n
    cap = "" if mi == args.max_iter else f", each capped at {mi} iterations"
    rows = "" if n_sub == data.n else f", on the first {n_sub} of {data.n} rows (rate scaled by {scale:.4g})"
    return {"value": its / dt * scale, "unit": "iterations/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"one fit of each variant{cap}{rows} ({its} iterations, {dt:.1f} s), C oracle, OpenMP threads"}


# ----------------------------------------------------------------- our arm
def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import _lib
    from paper_2107_04074_b200.engine import DeviceCorpus, run
    from paper_2107_04074_b200.seeding import SeedConfig, make_centroids

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    data, gen_s = load_workload(args)
    variants = args.variants.split(",")
    k = args.k
    from paper_2107_04074_b200.seeding import uniform_rows
    seed_rows = uniform_rows(data.n, k, args.seed)
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

    def fit_all(corpus_, tag=None):
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
            last = r
        return its, sims, nk, per, last

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
                its, sims, nk, per, _ = fit_all(corpus)
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
    # every step: the CSR shard's host arrays are staged in pinned memory and
    # uploaded (raw rows H2D; device-order layout, term renumbering and
    # float32 conversion rebuilt on the GPU) into the serving buffers of a
    # persistent DeviceCorpus, then the user's call spk.run(...) per variant
    # (seed row ids H2D, stats + assignments D2H).  W untimed warm-up steps
    # fill the engine cache for that corpus and capture its fit graphs.
    e2e_times, h2d, d2h = [], 0, 0
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
    del c
    e2e_ms = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_val = its_tot / (float(e2e_ms.item()) / 1e3)

    # ---- instrumented pass: per-entry-point event times -> roofline ----
    roof = roofline(args, data, corpus, dev, world)

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
            "e2e": {"value": e2e_val, "unit": "iterations/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof,
            "clocks": clocks}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, data)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline(args, data, corpus, dev, world):
    """Time every entry point with CUDA events over one step; bytes from SURVEY.md §8(d)."""
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
    kp = (k + 7) // 8 * 8
    with prof:
        for v in args.variants.split(","):
            prof.tag = v
            comm = Exchange.for_corpus(k, corpus, dev) if world > 1 else None
            r = run(data, k, v, SeedConfig(seed=args.seed), max_iter=args.max_iter, device=dev, corpus=corpus,
                    comm=comm, n_total=data.n)
            its = r.iterations
            ku = (k + 3) // 4 * 4
            csr_full = 8 * nnz + 8 * n + 4 * n          # indices+values, indptr, row eps
            # full passes: iteration 1 of every variant and every Lloyd iteration
            n_full = 1 + (len(its) - 1 if v == "standard" else 0)
            init_w = 8 * n + (4 * k * n if v in ("elkan", "simp_elkan") else 4 * n if "hamerly" in v else 0)
            lloyd_w = 4 * n
            b = csr_full * n_full + init_w + lloyd_w * (n_full - 1)
            bytes_by[("spkm_full_assign", v)] = b
            # center-row bytes the gather passes read through L1/L2 (4 kp per nnz)
            gather_by[("spkm_full_assign", v)] = 4 * kp * nnz * n_full
            if v in ("hamerly", "simp_hamerly"):
                bytes_by[("spkm_hamerly_bounds", v)] = 24 * n * (len(its) - 1)
                bytes_by[("spkm_hamerly_tighten", v)] = sum(8 * s.nnz_tighten + 24 * s.survivors for s in its[1:])
                bytes_by[("spkm_hamerly_rescan", v)] = sum(8 * s.nnz_rescan + 24 * s.survivors2 for s in its[1:])
                gather_by[("spkm_hamerly_rescan", v)] = sum(4 * kp * s.nnz_rescan for s in its[1:])
            if v in ("elkan", "simp_elkan"):
                b_bounds = (8 * ku + 16) * n * (len(its) - 1)
                b_scan = sum(8 * s.nnz_elkan + (8 * ku + 16) * s.survivors for s in its[1:])
                bytes_by[("spkm_elkan_bounds", v)] = b_bounds
                bytes_by[("spkm_elkan_scan", v)] = b_scan
                # the fused entry point (bound update + scan in one pass) moves both
                bytes_by[("spkm_elkan_bounds_scan", v)] = b_bounds + b_scan
            # center update (reported beside B_iter): 16 B of
            # int64 atomics per moved nnz; 20 B per (touched cluster, term)
            # to renormalise and take the drift
            bytes_by[("spkm_apply_moves", v)] = sum(16 * s.nnz_moved for s in its[1:])
            bytes_by[("spkm_move_centers", v)] = sum(20 * s.touched * data.dim for s in its)
            if dense:
                # tensor-core pass: 3 tf32 MMAs per (row, padded center, dim)
                kpad = (k + 255) // 256 * 256
                D = corpus.dense_dim
                rows = n * n_full + (sum(s.survivors for s in its[1:]) if "hamerly" in v else 0)
                flops_by[("spkm_dense_assign", v)] = 6 * rows * kpad * D
    torch.cuda.synchronize()
    times = prof.times_ms()
    calls = {}
    for (name, tag), ms in times.items():
        calls.setdefault(name, [0.0, 0])
        calls[name][0] += ms
    for name, e0, e1, tag in prof.records:
        calls[name][1] += 1
    total = sum(v[0] for v in calls.values())
    share = {nm: round(v[0] / total, 4) for nm, v in sorted(calls.items(), key=lambda x: -x[1][0])}
    # dominant KERNEL: the largest single-kernel entry point with a byte (HBM)
    # or flop (tensor) model; multi-kernel entry points (center update:
    # 4-5 short kernels whose event span includes host launch gaps in this
    # eager profiling pass) are reported beside it
    multi = {"spkm_move_centers", "spkm_center_thresholds", "spkm_aggregate_sums"}
    cand = [nm for nm in share if nm not in multi and any(key[0] == nm for key in list(bytes_by) + list(flops_by))]
    dom = cand[0] if cand else None
    out = {"bound": "hbm", "peak": pk.get("hbm_gbs"), "unit": "GB/s", "peak_source": src,
           "time_share": share, "traffic": None}
    if dom and any(key[0] == dom for key in flops_by):
        ms = calls[dom][0]
        f = sum(val for key, val in flops_by.items() if key[0] == dom)
        peak_tf32, how = tf32_peak(dev)
        ach = f / (ms / 1e3) / 1e12
        out.update({"bound": "tensor", "unit": "TFLOP/s", "kernel": dom, "achieved": ach, "peak": peak_tf32,
                    "peak_source": how, "frac": ach / peak_tf32, "launches": calls[dom][1],
                    "algorithmic_flops": f, "kernel_ms": ms,
                    "note": "3xTF32 flops (3 MMAs per product) over the kernel's CUDA-event time"})
    elif dom:
        ms = calls[dom][0]
        b = sum(val for key, val in bytes_by.items() if key[0] == dom)
        ach = b / (ms / 1e3) / 1e9
        out.update({"kernel": dom, "achieved": ach, "frac": ach / pk.get("hbm_gbs"), "launches": calls[dom][1],
                    "algorithmic_bytes": b, "kernel_ms": ms})
    tr = ncu_traffic(dom)
    if tr is not None:
        out["traffic"] = tr["dram_bytes_per_launch"]
        out["traffic_source"] = tr["source"]
        if "ncu_throughput_pct" in tr:
            out["ncu_throughput_pct"] = tr["ncu_throughput_pct"]
    # every entry point with a byte model: achieved GB/s of its event span
    per = {}
    for nm, (ms, nl) in calls.items():
        b = sum(val for key, val in bytes_by.items() if key[0] == nm)
        if b and ms:
            per[nm] = {"launches": nl, "ms": round(ms, 4), "algorithmic_bytes": b,
                       "achieved_gbs": round(b / (ms / 1e3) / 1e9, 1),
                       "frac": round(b / (ms / 1e3) / 1e9 / pk.get("hbm_gbs"), 4)}
    out["per_entry"] = per
    # the gather passes are bound by L1/L2 (ncu_throughput_pct), not HBM: the
    # center-row bytes they pull per second, beside the HBM view above
    gv = {}
    for nm, (ms, nl) in calls.items():
        g = sum(val for key, val in gather_by.items() if key[0] == nm)
        if g and ms:
            gv[nm] = {"center_row_bytes": g, "ms": round(ms, 4), "achieved_gbs": round(g / (ms / 1e3) / 1e9, 1)}
    if gv:
        out["center_gather"] = gv
    if "spkm_move_centers" in calls:
        b = sum(val for key, val in bytes_by.items() if key[0] == "spkm_move_centers")
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


def ncu_traffic(kernel_entry):
    """dram bytes per launch of the entry point's main kernel from a committed ncu --set full capture."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if kernel_entry is None or not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel_entry)
    except Exception:
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
