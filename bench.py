#!/usr/bin/env python
"""bench.py -- headline benchmark: BASELINE config 1 sketch of [A, b].

Workload (BASELINE.json configs[1]): dense fp64 A, n = 4,194,304 x d = 512,
b = A x* + 0.01 N(0,1); CountSketch to s = 8192 rows (hash buckets / signs
from seed) followed by the Gaussian projection 8192 -> 2048, i.e. the
reference's combined sketch of lsr_sketched's stacked [A, b]
(src/regression.cpp:76-79, src/sketch.cpp:108-123). Rows are sharded across
ranks (one GPU each); the count stage is local, its 8192 x 513 partial is
summed with NCCL allreduce inside the library, the Gaussian stage follows.

A "step" = one sketch_rows call over the whole (sharded) [A, b].
  value  : GB/s of [A, b] read, whole job, inputs resident in HBM
  e2e    : same metric through the public API with pinned HOST buffers
           (H2D of every row + D2H of the 2048 x 513 result inside the timing)
  roofline: the dominant kernel (count-sketch gather-reduce) vs measured HBM
  cpu_baseline: the oracle's reference-faithful single-thread count sketch
           loop + single-thread fp64 Gaussian stage on a bounded row sample.

`--impl reference` times the reference's CPU path (the oracle port: the
reference itself cannot be built here, Eigen3 is absent) with all host
threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ROWS, D_COLS, S_CS, S_FINAL = 4_194_304, 512, 8192, 2048
MASTER_SEED = 42


def derive_seed(seed: int, stream: int) -> int:
    m = (1 << 64) - 1
    s = seed ^ ((0x6A09E667F3BCC909 + stream * 0x9E3779B97F4A7C15) & m)
    z = (s + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


DATA_SEED = derive_seed(MASTER_SEED, 101)
OP_SEED = derive_seed(MASTER_SEED, 201)
STAGE2_SEED = derive_seed(OP_SEED, 1)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          "Active" in s[3 + i] and "Not" not in s[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_baseline_run(sample_rows: int, threads: int, reps: int = 1):
    """Reference CPU path on a bounded sample: count sketch of [A, b] (oracle C
    loop, sequential order) + the fp64 Gaussian stage 8192 -> 2048 (BLAS).
    Returns (GB/s of [A, b] read for the FULL workload extrapolated from the
    sample, seconds per sample step, description)."""
    from oracle import oracle as orc
    from threadpoolctl import threadpool_limits

    rng = np.random.default_rng(DATA_SEED & 0xFFFFFFFF)
    a = rng.standard_normal((sample_rows, D_COLS))
    xs = rng.standard_normal(D_COLS)
    b = a @ xs + 0.01 * rng.standard_normal(sample_rows)
    g = orc.gaussian_matrix(S_CS, S_FINAL, STAGE2_SEED) / np.sqrt(S_FINAL)  # operator draw: not timed
    t_count, t_gauss = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        mid = orc.count_sketch_rows(a, S_CS, OP_SEED, extra=b, threads=threads)
        t1 = time.perf_counter()
        with threadpool_limits(limits=threads):
            out = g.T @ mid
        t2 = time.perf_counter()
        t_count.append(t1 - t0)
        t_gauss.append(t2 - t1)
        assert out.shape == (S_FINAL, D_COLS + 1)
    tc, tg = min(t_count), min(t_gauss)
    full_bytes = N_ROWS * (D_COLS + 1) * 8
    full_time = tc * (N_ROWS / sample_rows) + tg
    desc = (f"{sample_rows} of {N_ROWS} rows of [A,b] fp64 ({sample_rows * (D_COLS + 1) * 8 / 1e9:.2f} GB): "
            f"count sketch {tc:.3f} s (oracle C loop, {threads} thread(s)) + Gaussian stage {tg:.3f} s "
            f"(numpy/OpenBLAS, {threads} thread(s)); full-size time extrapolated linearly in rows")
    return full_bytes / full_time / 1e9, tc + tg, desc


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    sample = args.cpu_sample_rows
    for _ in range(args.warmup):
        cpu_baseline_run(min(sample, 65536), threads)
    vals, secs = [], []
    desc = ""
    for _ in range(args.steps):
        v, s, desc = cpu_baseline_run(sample, threads)
        vals.append(v)
        secs.append(s)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "sketch GB/s of [A,b] read (CountSketch 8192 -> Gaussian 2048)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.median(secs)) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded N(0,1), b = A x* + 0.01 N(0,1))",
        "config": {"workload": "cfg1: combined sketch of [A,b], n=4194304, d=512, s=8192 -> 2048", "n": N_ROWS,
                   "d": D_COLS, "s_cs": S_CS, "s": S_FINAL},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def ncu_traffic_from_profiles():
    """dram bytes (read + write) per launch of the gather kernel from the
    committed ncu --set full summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_cs_gather_r01.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                return json.load(f).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1505_07570_b200 as rn

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", world_size=world, rank=rank,
                                device_id=torch.device("cuda", local))
        idl = [rn.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(idl, src=0)
        ctx = rn.Context(local, world, rank, idl[0])
    else:
        ctx = rn.Context(local)

    n_total = args.rows
    r0, r1 = rn.shard_rows(n_total, world, rank)
    n_loc = r1 - r0
    d = D_COLS
    gen = torch.Generator(device="cuda")
    gen.manual_seed((DATA_SEED + rank) & 0x7FFFFFFFFFFFFFFF)
    A = torch.randn(n_loc, d, dtype=torch.float64, device="cuda", generator=gen)
    xg = torch.Generator(device="cuda")
    xg.manual_seed(DATA_SEED & 0x7FFFFFFF)
    xstar = torch.randn(d, dtype=torch.float64, device="cuda", generator=xg)
    b = A @ xstar + 0.01 * torch.randn(n_loc, dtype=torch.float64, device="cuda", generator=gen)
    out = torch.empty(S_FINAL, d + 1, dtype=torch.float64, device="cuda")
    spec = rn.SketchSpec.combined(S_CS, rn.SketchSpec.gaussian(S_FINAL, STAGE2_SEED), OP_SEED)
    count_spec = rn.SketchSpec.count_sketch(S_CS, OP_SEED)
    mid = torch.empty(S_CS, d + 1, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream)
    torch.cuda.synchronize()

    def step():
        rn.sketch_rows(A, spec, extra=b, row_offset=r0, out=out, ctx=ctx)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (plans + Gaussian operator are built and cached here: operator generation is not timed)
    t_op = time.perf_counter()
    for _ in range(max(args.warmup, 1)):
        step()
    ctx.synchronize()
    t_op = time.perf_counter() - t_op

    # ---- timed region: K steps, device events on the library stream ----
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = ctx.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_bytes = n_total * (d + 1) * 8
    value = total_bytes / (ms * 1e-3) / 1e9

    # ---- dominant kernel: count-sketch gather-reduce timed alone (count-only call) ----
    for _ in range(2):
        rn.sketch_rows(A, count_spec, extra=b, row_offset=r0, out=mid, ctx=ctx)
    ctx.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kreps = max(3, args.steps)
    k0.record(stream)
    for _ in range(kreps):
        rn.sketch_rows(A, count_spec, extra=b, row_offset=r0, out=mid, ctx=ctx)
    k1.record(stream)
    k1.synchronize()
    k_ms = k0.elapsed_time(k1) / kreps
    alg_bytes = n_loc * (d + 1) * 8 + S_CS * (d + 1) * 8
    peak, peak_kind = load_peaks()
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty(n_loc, d, dtype=torch.float64).pin_memory()
        bh = torch.empty(n_loc, dtype=torch.float64).pin_memory()
        Ah.copy_(A)
        bh.copy_(b)
        outh = np.empty((S_FINAL, d + 1), dtype=np.float64)
        rn.sketch_rows(Ah, spec, extra=bh, row_offset=r0, out=outh, ctx=ctx)  # warm
        barrier()
        e_steps = max(1, args.e2e_steps)
        t0 = time.perf_counter()
        for _ in range(e_steps):
            rn.sketch_rows(Ah, spec, extra=bh, row_offset=r0, out=outh, ctx=ctx)
        barrier()
        es = (time.perf_counter() - t0) / e_steps
        if world > 1:
            t = torch.tensor([es], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            es = float(t.item())
        same = np.array_equal(outh, out.cpu().numpy())
        e2e = {"value": total_bytes / es / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(n_total * (d + 1) * 8),
               "d2h_bytes_per_step": int(S_FINAL * (d + 1) * 8), "ms_per_step": es * 1e3,
               "matches_device_result_bitwise": bool(same)}
        del Ah, bh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, s, desc = cpu_baseline_run(args.cpu_sample_rows, 1)
        cpu = {"value": v, "unit": "GB/s", "cores": 1, "kind": "port", "sample": desc}

    if rank == 0:
        line = {
            "metric": "sketch GB/s of [A,b] read (CountSketch 8192 -> Gaussian 2048)",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) A on device, b = A x* + 0.01 N(0,1))",
            "config": {"workload": "cfg1: combined sketch of [A,b], n=4194304, d=512, s=8192 -> 2048",
                       "n": n_total, "d": d, "s_cs": S_CS, "s": S_FINAL, "parallelism": f"rows sharded x{world}",
                       "l2": "inputs (17.2 GB) larger than L2; no flush needed",
                       "operator_build_s": round(t_op, 3)},
            "roofline": {"bound": "hbm", "kernel": "cs_gather_kernel (count sketch gather-reduce)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic_from_profiles(),
                         "alg_bytes_per_launch": alg_bytes, "kernel_ms": k_ms,
                         "frac_of_8TBs_nominal": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=N_ROWS)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample-rows", type=int, default=1 << 20)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
