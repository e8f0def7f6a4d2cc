#!/usr/bin/env python3
"""FiGaRo B200 benchmark: input tuples/s to compute R (FP64).

One step = one full pipeline over the configured database (grouping sort,
counts, heads/tails, TSQR, sign-normalised R) from device-resident shuffled
relations.  The default workload is C3 at scale 1.0 (101 M input tuples, the
largest BASELINE config); `--config C1..C5` selects another.

N>1 (torchrun): `--scaling weak` (default) gives every rank a full-size
database over its own key range; `--scaling strong` generates ONE global
database and shards it through the real partitioner
(paper_2204_00525_b200/distributed.py: key-hash sharding, heavy-key splitting,
count all-reduce, R3 summary exchange).  Per-rank R factors are all-gathered
over NCCL and merged by one more device TSQR.

`--impl reference` times the reference's own CPU implementation: the
unmodified reference run_pipeline (oracle/_ref/figaro_ref, compiled from
/root/reference) with all host threads, on the same workload at the
reference scale (REF_SCALE: 1.0 except C3, whose reference needs ~1.7 KB of
host RAM and ~2.5 us of CPU per fact row; it runs at 0.1).  The database is
canonicalised once and run_pipeline is repeated in-process.  The GPU arm
reports its own tuples/s at exactly that scale as `at_reference_scale`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "input tuples/sec to compute R (FP64)"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "figaro_ref")
REF_SCALE = {"C1": 1.0, "C2": 1.0, "C3": 0.1, "C4": 1.0, "C5": 1.0}
TREES = {"C1": "R1(R2)", "C2": "R1(R2)", "C3": "D1(F(D2,D3))", "C4": "R1(R2(R3))",
         "C5": "R1(R2)"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """FP64 tensor (DMMA, mma.sync m8n8k4 f64) peak measured by
    scripts/fp64_peak.cu on a B200 of this pool; MEASURED_PEAKS.json has no
    FP64 entry."""
    p = os.path.join(ROOT, "profiles", "fp64_peak_r1.json")
    try:
        with open(p) as f:
            return float(json.load(f)["dmma_tflops"]), \
                "builder-measured DMMA (profiles/fp64_peak_r1.json; not in MEASURED_PEAKS.json)"
    except Exception:
        return 37.0, "datasheet fallback"


def ncu_traffic(config: str, scale: float):
    """DRAM bytes per launch of the heads/tails launches from the committed
    `ncu --set full` capture of this config (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"{config}@{scale:g}")
        if e:
            return e["headtail_dram_bytes_per_launch"], e["source"]
    except Exception:
        pass
    return None, None


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML during the timed
    region (no subprocess: forking a multi-GB process stalls the host)."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def run(self):
        nv = self.nv
        while nv is not None and not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            self.stop.wait(0.02)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        nv = self.nv
        reasons = sorted({name for _, rs in self.samples for name, attr in self.REASONS
                          if rs & getattr(nv, attr, 0)})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "nvml"}


# ------------------------------------------------------------ reference arm


def reference_runs(config: str, scale: float, seed: int, reps: int, budget: float):
    """The unmodified reference run_pipeline (oracle/_ref/figaro_ref --repeat):
    database canonicalised once, run_pipeline timed `reps` times (stopping
    once `budget` seconds of pipeline time are spent).  Returns (seconds per
    run, input rows, cores, canonicalize seconds) or None."""
    from paper_2204_00525_b200 import fgdb, workloads
    if not os.path.exists(REF_BIN):
        return None
    db = workloads.make(config, seed=seed, scale=scale)
    rows = workloads.input_rows(db)
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "db.fgdb")
        fgdb.write_fgdb(p, db)
        del db
        out = subprocess.run([REF_BIN, "run", p, p + ".rs", "--threads", str(cores),
                              "--repeat", str(max(1, reps)), "--budget", str(budget)],
                             capture_output=True, text=True, check=True).stdout
    secs, canon = [], 0.0
    for line in out.splitlines():
        kv = dict(x.split("=") for x in line.split() if "=" in x)
        if line.startswith("rep="):
            secs.append(float(kv["pipeline"]))
        elif line.startswith("ok"):
            canon = float(kv["canon"])
            if not secs:
                secs.append(float(kv["pipeline"]))
    return secs, rows, cores, canon


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    scale = args.scale * (args.ref_scale if args.ref_scale else REF_SCALE[args.config])
    warm = min(args.warmup, 1)  # a CPU pipeline needs one warm run at most
    res = reference_runs(args.config, scale, args.seed, warm + args.steps, args.ref_budget)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/figaro_ref not built"}))
        return
    secs, rows, cores, canon = res
    timed = secs[warm:] or secs
    t = statistics.median(timed)
    v = rows / t
    sample = (f"{args.config} at scale {scale:g} ({rows} input rows, seed {args.seed}), full "
              f"database; reference run_pipeline(assume_reduced) repeated in-process on the "
              f"once-canonicalised relations ({len(timed)} timed runs after {warm} warm-up, "
              f"median; budget {args.ref_budget:g} s; canonicalize {canon:.2f} s excluded)")
    line = {"metric": METRIC, "value": v, "unit": "tuples/s", "n_gpus": args.gpus,
            "steps": len(timed), "steps_requested": args.steps, "warmup": warm,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "scale": scale, "input_rows": rows,
                       "tree": TREES[args.config]},
            "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------ GPU arm


def device_relations(db, F, torch):
    return [F.Relation(r.name, r.key_attrs, r.data_attrs, torch.from_numpy(r.keys).cuda(),
                       torch.from_numpy(r.data).cuda()) for r in db.relations]


class Runner:
    """One database on the device; step() = one pipeline (+ gather/merge)."""

    def __init__(self, db, F, D, torch, local, world, presorted=False, plan=None, heavy=None):
        self.F, self.D, self.torch, self.local, self.world = F, D, torch, local, world
        self.rels = device_relations(db, F, torch)
        self.tree = F.build_join_tree(self.rels, db.root, db.parent)
        self.root = db.root
        self.n = sum(len(r.data_attrs) for r in db.relations)
        # Strong scaling: the partition plan and this rank's heavy-key rows
        # (device-resident); shards with replicated rows need reduction.
        self.plan = plan
        self.heavy = None
        if heavy is not None:
            self.heavy = [(k, torch.from_numpy(d).cuda()) for k, d in heavy]
        reduced = plan is None or not plan.needs_reduction(db.relations)
        self.opts = F.PipelineOptions(assume_reduced=reduced)
        self.rows = sum(r.rows for r in db.relations) + \
            sum(int(k.shape[0]) for k, _ in (heavy or []))
        self.gather_s = 0.0
        if presorted:
            # Paper convention: relations already sorted by
            # key; permute them once with the pipeline's own sort order.
            F.run_pipeline(self.rels, self.tree, self.opts, device=local, fetch_counts=False)
            for i, r in enumerate(self.rels):
                perm = torch.from_numpy(F.fetch_permutation(i, r.row_count(), local)).long().cuda()
                self.rels[i] = F.Relation(r.name, r.key_attrs, r.data_attrs,
                                          r.keys[perm].contiguous(), r.data[perm].contiguous())

    def step(self):
        if self.plan is not None and self.world > 1:
            # Strong scaling: the whole per-rank flow of distributed.py
            # (pipeline on the shard, heavy-key stage, gathers, merge).
            out = []
            g0 = time.perf_counter()
            R = self.D.distributed_factor(self.rels, self.heavy, self.tree, self.n, self.plan,
                                          self.root, device=self.local,
                                          assume_reduced=self.opts.assume_reduced, results=out)
            self.torch.cuda.synchronize()
            self.gather_s += time.perf_counter() - g0
            return (out[0] if out else _EmptyResult()), R
        res = self.F.run_pipeline(self.rels, self.tree, self.opts, device=self.local,
                                  fetch_counts=False)
        R = res.factor.r
        if self.world > 1:
            g0 = time.perf_counter()
            R = self.D.gather_and_merge(R, lambda p, n: self.D.device_merge(p, n, device=self.local))
            self.torch.cuda.synchronize()
            self.gather_s += time.perf_counter() - g0
        return res, R

    def timed(self, steps, warmup, stream, dist=None, clocks=None):
        torch = self.torch
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        acc = {"group": 0.0, "counts": 0.0, "figaro": 0.0, "post": 0.0, "ht_s": 0.0,
               "ts_s": 0.0, "ht_launches": 0, "ht_bytes": 0.0, "fused_flops": 0.0,
               "ts_flops": 0.0, "fused_launches": 0, "syncs": 0, "mallocs": 0}
        self.gather_s = 0.0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ctx = self.F.get_context(self.local)
        k0 = ctx.kernel_launches()
        cm = clocks if clocks is not None else _Null()
        with cm:
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                res, _ = self.step()
                acc["group"] += res.seconds_group
                acc["counts"] += res.seconds_counts
                acc["figaro"] += res.seconds_figaro
                acc["post"] += res.seconds_postprocess
                acc["ht_s"] += res.seconds_headtail_kernels
                acc["ts_s"] += res.seconds_tsqr_kernels
                acc["ht_launches"] += res.headtail_launches
                acc["ht_bytes"] += res.headtail_bytes
                acc["fused_flops"] += res.headtail_fused_flops
                acc["ts_flops"] += res.tsqr_stage_flops
                acc["fused_launches"] += res.fused_launches
                acc["syncs"] += res.host_syncs
                acc["mallocs"] += getattr(res, "device_mallocs", 0)
            e1.record(stream)
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
        acc["launches"] = ctx.kernel_launches() - k0
        ms = e0.elapsed_time(e1) / steps
        if dist is not None:
            t = torch.tensor([ms, self.gather_s / steps * 1e3], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, g = float(t[0]), float(t[1])
        else:
            g = 0.0
        acc["gather_ms"] = g
        return ms, {k: (v / steps if isinstance(v, float) else v) for k, v in acc.items()}


class _EmptyResult:
    """Phase counters of a rank whose shard join was empty."""
    seconds_group = seconds_counts = seconds_figaro = seconds_postprocess = 0.0
    seconds_headtail_kernels = seconds_tsqr_kernels = headtail_bytes = 0.0
    headtail_fused_flops = tsqr_stage_flops = 0.0
    headtail_launches = fused_launches = host_syncs = device_mallocs = 0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def roofline_objects(acc, steps, config, scale):
    """The heads/tails launches against measured HBM bandwidth and the TSQR
    stage against the measured FP64 tensor peak, each with the algorithmic
    units the library counted; the slower one first."""
    hbm, hsrc = load_peaks()
    fp64, fsrc = fp64_peak()
    launches = max(1, acc["ht_launches"] // steps)
    ht_s, ts_s = acc["ht_s"], acc["ts_s"]
    fused = acc["fused_launches"] // steps
    kernel = ("k_heads_tails_tsqr (fused own heads/tails -> TSQR leaf) x %d + k_heads_tails x %d"
              % (fused, launches - fused)) if fused else \
        "k_heads_tails (own heads/tails and project-away generalized heads/tails) x %d" % launches
    achieved = acc["ht_bytes"] / ht_s / 1e9 if ht_s > 0 else 0.0
    traffic, tsrc = ncu_traffic(config, scale)
    ht = {"kernel": kernel, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
          "frac": achieved / hbm, "traffic": traffic,
          "traffic_source": tsrc,
          "algorithmic_bytes_per_launch": acc["ht_bytes"] / launches,
          "launches_per_step": launches, "ms_per_launch": ht_s / launches * 1e3,
          "peak_source": hsrc,
          "fused_fp64": {"flops_per_step": acc["fused_flops"],
                         "achieved_tflops": acc["fused_flops"] / ht_s / 1e12 if ht_s > 0 else 0.0}}
    tfl = acc["ts_flops"] / ts_s / 1e12 if ts_s > 0 else 0.0
    ts = {"kernel": "TSQR stage (k_tsqr_warp / k_tsqr_la leaves of the unfused spans + merges "
                    "+ k_normalize)",
          "bound": "tensor", "achieved": tfl, "peak": fp64, "unit": "TFLOP/s", "frac": tfl / fp64,
          "traffic": None, "algorithmic_flops_per_step": acc["ts_flops"],
          "ms_per_step": ts_s * 1e3, "peak_source": fsrc}
    return (ht, ts) if ht_s >= ts_s else (ts, ht)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-side collectives, for checking the N>1 flow with "
                         "ranks sharing one GPU (no rank waits on another's kernels)")
    ap.add_argument("--ref-scale", type=float, default=None,
                    help="reference-arm scale relative to --scale (default REF_SCALE[config])")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="seconds of reference pipeline time per reference arm")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the reference-scale and pre-sorted GPU lines")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2204_00525_b200 import distributed as D
    from paper_2204_00525_b200 import figaro as F
    from paper_2204_00525_b200 import workloads

    if args.dist_backend == "gloo":  # ranks may share a GPU
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    stream = torch.cuda.current_stream()
    ctx = F.get_context(local)
    ctx.bind_current_stream()
    dd = dist if world > 1 else None

    plan = heavy = None
    if world > 1 and args.scaling == "strong":
        # One global database through the partition plan (distributed.py).
        full = workloads.make(args.config, seed=args.seed, scale=args.scale)
        plan = D.plan_partition(full.relations, full.root, world, parent=full.parent)
        db = D.shard_database(full, rank, world, plan)
        heavy = D.heavy_rows(full.relations, plan, rank) if plan.combine else None
        global_rows = workloads.input_rows(full)
        del full
    else:
        db = D.weak_shard(workloads.make(args.config, seed=args.seed + 1000003 * rank,
                                         scale=args.scale), rank, world)
    runner = Runner(db, F, D, torch, local, world, plan=plan, heavy=heavy)
    m_rank = runner.rows
    clk = ClockSampler(local)
    ms, acc = runner.timed(args.steps, args.warmup, stream, dd, clocks=clk)
    if plan is not None:
        m_total = float(global_rows)  # strong scaling: the one database's tuples
    elif world > 1:
        t = torch.tensor([m_rank], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        m_total = float(t.item())
    else:
        m_total = m_rank
    value = m_total / (ms * 1e-3)

    # e2e: host (pinned) relations through the same public API; H2D of the
    # step's inputs and D2H of R inside the timed region.
    host_rels, pinned, h2d = [], [], 0
    for r in db.relations:
        k = torch.from_numpy(r.keys).pin_memory()
        d = torch.from_numpy(r.data).pin_memory()
        pinned.append((k, d))
        h2d += k.numel() * 8 + d.numel() * 8
        host_rels.append(F.Relation(r.name, r.key_attrs, r.data_attrs, k.numpy(), d.numpy()))
    opts = runner.opts
    if heavy is not None:
        h2d += sum(d.size * 8 for _, d in heavy)

    def e2e_step():
        if plan is not None:  # strong scaling: the whole distributed flow from host buffers
            return D.distributed_factor(host_rels, heavy, runner.tree, runner.n, plan,
                                        runner.root, device=local,
                                        assume_reduced=opts.assume_reduced).cpu().numpy()
        hr = F.run_pipeline(host_rels, runner.tree, opts, device=local, fetch_counts=False)
        Rh = hr.factor.r
        if world > 1:
            Rh = D.gather_and_merge(torch.from_numpy(Rh).cuda(),
                                    lambda p, n: D.device_merge(p, n, device=local)).cpu().numpy()
        return Rh

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    n = sum(len(r.data_attrs) for r in db.relations)
    e2e = {"value": m_total / e2e_s, "unit": "tuples/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": n * n * 8, "ms_per_step": e2e_s * 1e3}
    # The e2e bound: a plain pinned host -> device copy of the same bytes
    # (best of 3), i.e. the PCIe time no implementation can go below.
    dev_bufs = [(torch.empty_like(k, device="cuda"), torch.empty_like(d, device="cuda"))
                for k, d in pinned]
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        for (dk, dd_), (k, d) in zip(dev_bufs, pinned):
            dk.copy_(k, non_blocking=True)
            dd_.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - c0)
    del dev_bufs, pinned, host_rels
    h2d_gbs = h2d / best / 1e9
    e2e["roofline"] = {"bound": "pcie_h2d", "achieved": h2d / e2e_s / 1e9, "peak": h2d_gbs,
                       "unit": "GB/s", "frac": (h2d / e2e_s / 1e9) / h2d_gbs,
                       "peak_source": "measured here: pinned cudaMemcpyAsync of the step's "
                                      "input bytes, best of 3"}

    extras = {}
    if not args.no_extras and world == 1:
        # Paper convention: pre-sorted input, sort (group phase) excluded.
        del runner
        pre = Runner(db, F, D, torch, local, world, presorted=True)
        pms, pacc = pre.timed(max(3, args.steps // 2), args.warmup, stream)
        excl = pms - pacc["group"] * 1e3
        extras["paper_convention"] = {
            "value": m_total / (excl * 1e-3), "ms_per_step": excl,
            "note": "relations pre-sorted by key (PAPER.md:951-954); group phase time excluded"}
        del pre
        rs = args.scale * (args.ref_scale if args.ref_scale else REF_SCALE[args.config])
        if rs != args.scale:
            sdb = workloads.make(args.config, seed=args.seed, scale=rs)
            srun = Runner(sdb, F, D, torch, local, world)
            sms, _ = srun.timed(args.steps, args.warmup, stream)
            extras["at_reference_scale"] = {"scale": rs, "input_rows": srun.rows,
                                            "value": srun.rows / (sms * 1e-3), "ms_per_step": sms}
            del srun, sdb

    if rank == 0:
        roof, other = roofline_objects(acc, args.steps, args.config, args.scale)
        line = {
            "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded N(0,1), Zipf keys, shuffled rows; inputs > L2, no flush "
                    "needed)",
            "config": {"workload": args.config, "scale": args.scale,
                       "input_rows": int(m_total), "input_rows_per_gpu": m_rank,
                       "columns": n, "tree": TREES[args.config],
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": (f"grid {plan.attrs}x{plan.dims}, {len(plan.combine)} "
                                       f"combined / {len(plan.heavy)} split heavy keys (strong)"
                                       if plan is not None else
                                       f"key-hash x{world}" + (" (weak)" if world > 1 else "")),
                       "reference_scale": args.scale * (args.ref_scale or REF_SCALE[args.config])},
            "phases_ms": {"group": acc["group"] * 1e3, "counts": acc["counts"] * 1e3,
                          "figaro": acc["figaro"] * 1e3, "post": acc["post"] * 1e3,
                          "gather": acc["gather_ms"]},
            "host_syncs_per_step": acc["syncs"] // args.steps,
            "device_mallocs_in_timed_steps": acc["mallocs"],
            "roofline": roof, "roofline_other": other,
            "e2e": e2e, "gpu_launches": acc["launches"], "clocks": clk.summary(),
        }
        line.update(extras)
        if not args.no_cpu_baseline and world == 1:
            rs = args.scale * (args.ref_scale or REF_SCALE[args.config])
            cb = reference_runs(args.config, rs, args.seed, 1, 0.0)
            if cb:
                secs, rows, cores, canon = cb
                line["cpu_baseline"] = {
                    "value": rows / secs[0], "unit": "tuples/s", "cores": cores,
                    "kind": "reference",
                    "sample": f"{args.config} at scale {rs:g} ({rows} input rows, seed "
                              f"{args.seed}); one reference run_pipeline(assume_reduced) on "
                              f"{cores} threads, canonicalize ({canon:.2f} s) excluded"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
