#!/usr/bin/env python3
"""FiGaRo B200 benchmark: input tuples/s to compute R (FP64).

One step = one full pipeline over the configured database (grouping sort,
counts, heads/tails, TSQR, sign-normalised R) from device-resident shuffled
relations; for N>1 each rank owns a key-hash shard (weak scaling: a rank's
shard is a full-size config over its own key range) and the per-rank R
factors are all-gathered over NCCL and merged by one more device TSQR.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/figaro_ref, compiled from /root/reference) on a bounded sample of
the same workload, with all host threads.
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

# Algorithmic units of the dominant kernel, the own-group
# heads/tails kernel of each relation (fused with the TSQR leaf when the
# relation has <= 32 data columns): input rows read once through the sort
# permutation (8 B per element + 4 B of permutation per row), heads written
# once, tails written once only when not fused.  FP64 work of the fused
# kernel: the TSQR flops of the own-tails spans, 2 m w^2 - 2/3 w^3.


def _groups(r) -> int:
    return np.unique(r.keys, axis=0).shape[0] if r.keys.shape[1] else 1


def headtail_units(db):
    bytes_, flops = 0, 0.0
    for r in db.relations:
        w = len(r.data_attrs)
        g = _groups(r)
        fused = 0 < w <= 32
        bytes_ += 8 * r.rows * w + 4 * r.rows + 8 * g * w
        if not fused:
            bytes_ += 8 * (r.rows - g) * w
        m = r.rows - g
        if fused and m > 0:
            flops += 2.0 * m * w * w - 2.0 / 3.0 * w ** 3
    return bytes_, flops


def tsqr_flops(db) -> float:
    """2 m w^2 - 2/3 w^3 per column span + 2/3 N^3 per final merge,
    for 2-relation same-key trees: own tails of each relation + final block."""
    ncols = sum(len(r.data_attrs) for r in db.relations)
    fl = 0.0
    for r in db.relations:
        w = len(r.data_attrs)
        m = r.rows - _groups(r)
        fl += 2.0 * m * w * w - 2.0 / 3.0 * w ** 3
    groot = _groups(db.relations[db.root])
    fl += 2.0 * groot * ncols ** 2 - 2.0 / 3.0 * ncols ** 3
    fl += 2.0 / 3.0 * ncols ** 3
    return fl


def fp64_peak(kind: str = "dfma"):
    p = os.path.join(ROOT, "profiles", "fp64_peak_r1.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return (float(d[f"{kind}_tflops"]),
                f"measured (profiles/fp64_peak_r1.json, {kind.upper()}; not in MEASURED_PEAKS.json)")
    except Exception:
        return 37.0, "datasheet fallback"


def ncu_traffic(prefix: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_traffic_r1.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic_r1.json")
    try:
        with open(p) as f:
            d = json.load(f)
        for k, v in d.items():
            if prefix in k:
                return v["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


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


def shard_database(config: str, scale: float, seed: int, rank: int, world: int):
    """Rank r's shard: the config generated with its own seed, keys moved to
    the key range of hash bucket r (a key-hash partition of a world-times
    larger database; every key group stays on one GPU)."""
    from paper_2204_00525_b200 import workloads
    db = workloads.make(config, seed=seed + 1000003 * rank, scale=scale)
    if world > 1:
        for r in db.relations:
            if r.keys.size:
                r.keys = r.keys * world + rank
    return db


def cpu_reference(config: str, scale: float, seed: int, sample_scale: float, steps: int):
    """Runs oracle/_ref/figaro_ref (the unmodified reference run_pipeline) on a
    bounded sample; returns (tuples/s per run list, sample rows, cores, desc)."""
    from paper_2204_00525_b200 import fgdb, workloads
    if not os.path.exists(REF_BIN):
        return None
    db = workloads.make(config, seed=seed, scale=scale * sample_scale)
    rows = workloads.input_rows(db)
    cores = os.cpu_count() or 1
    vals = []
    canon = []
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "sample.fgdb")
        fgdb.write_fgdb(p, db)
        for _ in range(steps):
            out = subprocess.run([REF_BIN, "run", p, p + ".rs", "--threads", str(cores)],
                                 capture_output=True, text=True, check=True).stdout
            kv = dict(x.split("=") for x in out.split() if "=" in x)
            vals.append(rows / float(kv["pipeline"]))
            canon.append(float(kv["canon"]))
    desc = (f"{config} at scale {scale * sample_scale:g} ({rows} input rows, seed {seed}); "
            f"reference run_pipeline(assume_reduced) wall time, canonicalize excluded "
            f"(median {statistics.median(canon):.2f} s extra)")
    return vals, rows, cores, desc


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    res = cpu_reference(args.config, args.scale, args.seed, args.ref_sample, args.steps + args.warmup)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/figaro_ref not built"}))
        return
    vals, rows, cores, desc = res
    timed = vals[args.warmup:] or vals
    v = statistics.median(timed)
    line = {"metric": METRIC, "value": v, "unit": "tuples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": rows / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "scale": args.ref_sample * args.scale,
                       "tree": "R1(R2)"},
            "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": cores, "kind": "reference",
                             "sample": desc},
            "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--ref-sample", type=float, default=1.0 / 16)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2204_00525_b200 import figaro as F

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = F.get_context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    db = shard_database(args.config, args.scale, args.seed, rank, world)
    m_rank = sum(r.rows for r in db.relations)
    rels = [F.Relation(r.name, r.key_attrs, r.data_attrs, torch.from_numpy(r.keys).cuda(),
                       torch.from_numpy(r.data).cuda()) for r in db.relations]
    tree = F.build_join_tree(rels, db.root, db.parent)
    n = sum(len(r.data_attrs) for r in db.relations)
    opts = F.PipelineOptions(assume_reduced=True)

    from paper_2204_00525_b200 import distributed as D
    merge = lambda parts, nn: D.device_merge(parts, nn, device=local)  # noqa: E731

    def step():
        res = F.run_pipeline(rels, tree, opts, device=local, fetch_counts=False)
        R = D.gather_and_merge(res.factor.r, merge) if world > 1 else res.factor.r
        return res, R

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    k0 = ctx.kernel_launches()
    phases = {"group": 0.0, "counts": 0.0, "figaro": 0.0, "post": 0.0}
    kern = {"headtail": 0.0, "tsqr": 0.0, "headtail_launches": 0}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            res, R = step()
            phases["group"] += res.seconds_group
            phases["counts"] += res.seconds_counts
            phases["figaro"] += res.seconds_figaro
            phases["post"] += res.seconds_postprocess
            kern["headtail"] += res.seconds_headtail_kernels
            kern["tsqr"] += res.seconds_tsqr_kernels
            kern["headtail_launches"] += res.headtail_launches
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = ctx.kernel_launches() - k0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = m_rank * world / (ms * 1e-3)

    # e2e: host (pinned) relations through the same public API; H2D of the
    # step's inputs and D2H of R inside the timed region.
    host_rels = []
    pinned = []
    h2d = 0
    for r in db.relations:
        k = torch.from_numpy(r.keys).pin_memory()
        d = torch.from_numpy(r.data).pin_memory()
        pinned.append((k, d))
        h2d += k.numel() * 8 + d.numel() * 8
        host_rels.append(F.Relation(r.name, r.key_attrs, r.data_attrs, k.numpy(), d.numpy()))
    F.run_pipeline(host_rels, tree, opts, device=local, fetch_counts=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        hr = F.run_pipeline(host_rels, tree, opts, device=local, fetch_counts=False)
        Rh = hr.factor.r
        if world > 1:
            Rh = D.gather_and_merge(torch.from_numpy(Rh).cuda(), merge).cpu().numpy()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": m_rank * world / e2e_s, "unit": "tuples/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": n * n * 8, "ms_per_step": e2e_s * 1e3}
    # The e2e roofline: a plain pinned host -> device copy of the same bytes
    # (best of 3), i.e. the PCIe time no implementation can go below.
    dev_bufs = [(torch.empty_like(k, device="cuda"), torch.empty_like(d, device="cuda"))
                for k, d in pinned]
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        for (dk, dd), (k, d) in zip(dev_bufs, pinned):
            dk.copy_(k, non_blocking=True)
            dd.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - c0)
    del dev_bufs
    h2d_gbs = h2d / best / 1e9
    e2e["roofline"] = {"bound": "pcie_h2d", "achieved": h2d / e2e_s / 1e9, "peak": h2d_gbs,
                       "unit": "GB/s", "frac": (h2d / e2e_s / 1e9) / h2d_gbs,
                       "peak_source": "measured here: pinned cudaMemcpyAsync of the step's input bytes, best of 3"}

    if rank == 0:
        hbm, src = load_peaks()
        fp64, fsrc = fp64_peak()
        ht_bytes, ht_flops = headtail_units(db)
        launches_per_step = max(1, kern["headtail_launches"] // args.steps)
        ht_s = kern["headtail"] / args.steps          # per step (all launches)
        achieved = ht_bytes / ht_s / 1e9 if ht_s > 0 else 0.0
        line = {
            "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1), shuffled rows; inputs > L2, no flush needed)",
            "config": {"workload": args.config, "scale": args.scale, "input_rows_per_gpu": m_rank,
                       "columns": n, "tree": "R1(R2)" if len(db.relations) == 2 else "see workloads",
                       "l2": "inputs larger than L2 (no flush)", "parallelism": f"key-hash x{world}"},
            "phases_ms": {k: v / args.steps * 1e3 for k, v in phases.items()},
            "roofline": {"kernel": "k_heads_tails_tsqr (fused heads/tails -> TSQR leaf; "
                                   "k_heads_tails when w > 32)",
                         "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm,
                         "traffic": ncu_traffic("k_heads_tails_tsqr<2, WCfg<16")
                         if args.config == "C2" else None,
                         "traffic_source": "profiles/ncu_traffic_r1.json (ncu --set full, C2; summary in profiles/r1s2/ncu_fused_c2.txt)",
                         "algorithmic_bytes_per_launch": ht_bytes / launches_per_step,
                         "launches_per_step": launches_per_step,
                         "ms_per_launch": ht_s / launches_per_step * 1e3,
                         "peak_source": src},
            "roofline_fp64": {"kernel": "same launches, TSQR work of the own-tails spans",
                              "achieved": ht_flops / ht_s / 1e12 if ht_s > 0 else 0.0,
                              "peak": fp64, "unit": "TFLOP/s",
                              "frac": (ht_flops / ht_s / 1e12) / fp64 if ht_s > 0 else 0.0,
                              "peak_source": fsrc},
            "tsqr_stage": {"flops": tsqr_flops(db), "ms": kern["tsqr"] / args.steps * 1e3,
                           "note": "remaining TSQR work (final block, unfused spans, merges)"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        # When the TSQR stage (unfused wide spans, merges) takes longer than the
        # heads/tails launches, it is the dominant kernel: report it against
        # the measured FP64 tensor (DMMA) peak instead.
        ts_s = kern["tsqr"] / args.steps
        if ts_s > ht_s and len(db.relations) == 2:  # tsqr_flops: 2-relation trees
            dpk, dsrc = fp64_peak(kind="dmma")
            tfl = tsqr_flops(db) / ts_s / 1e12
            line["roofline_headtail"] = line["roofline"]
            line["roofline"] = {
                "kernel": "TSQR stage (k_tsqr_la look-ahead blocked TSQR + merges)",
                "bound": "tensor", "achieved": tfl, "peak": dpk, "unit": "TFLOP/s",
                "frac": tfl / dpk, "traffic": None,
                "algorithmic_flops_per_step": tsqr_flops(db), "ms_per_step": ts_s * 1e3,
                "peak_source": dsrc}
        if not args.no_cpu_baseline:
            cb = cpu_reference(args.config, args.scale, args.seed, args.ref_sample, 1)
            if cb:
                vals, rows, cores, desc = cb
                line["cpu_baseline"] = {"value": vals[0], "unit": "tuples/s", "cores": cores,
                                        "kind": "reference", "sample": desc}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
