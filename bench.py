"""GEEK end-to-end benchmark: bucketize + SILK + assign on synthetic
SIFT-like data (BASELINE.json configs[1]: 100M x 128 float32, E2LSH/rank-split
bucketing with m=40 tables of t=100,000 buckets, SILK with L=20, K=3,
delta=10, Euclidean one-pass assignment; g_logical=8 workers).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl geek|reference] [--n N]

One step = one full run_pipeline over the resident dataset (value) or,
for `e2e`, host pinned data -> H2D -> pipeline -> D2H of the labels.
Multi-GPU: one process per GPU (torchrun), points sharded contiguously,
total n fixed (strong scaling); time = max over ranks of CUDA-event time.
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

METRIC = "GEEK end-to-end points/sec (bucketize+SILK+assign), 128-d dense, 1/2/4/8 B200"
# t = n / points_per_bucket: buckets hold one planted cluster's worth of points
# (n / C), the ratio of the reference's config 1 (100K points, C = t = 100);
# K = 2 as in SURVEY config 3.  With SURVEY 8(d)'s t = n/1000, K = 3 no bin
# survives the vote at 100M and the run degenerates to the random fallback.
PARAMS = dict(d=128, clusters=1000, separation=10.0, m=40, points_per_bucket=100_000, L=20, K=2, delta=10, g=8,
              tseed=1, sseed=2, data_seed=0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="geek", choices=["geek", "reference"])
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=20_000)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU reference arm: the oracle port of the reference pipeline (test infra)

def cpu_reference(n_sample: int, steps: int, warmup: int):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    from oracle import geek_oracle as O

    P = PARAMS
    X, _ = O.gaussian_mixture(n_sample, P["d"], max(1, min(P["clusters"], n_sample // 100)), P["separation"],
                              P["data_seed"])
    t = max(2, n_sample // P["points_per_bucket"])
    times = []
    for i in range(max(0, warmup) + steps):
        t0 = time.perf_counter()
        O.pipeline_dense(X, P["m"], t, P["tseed"], P["K"], P["L"], P["delta"], P["sseed"], g=P["g"])
        el = time.perf_counter() - t0
        if i >= warmup:
            times.append(el)
    sec = float(np.mean(times))
    return dict(value=n_sample / sec, unit="points/s", cores=1, kind="port",
                sample=f"{n_sample} x {P['d']} gaussian-mixture (C={max(1, min(P['clusters'], n_sample // 100))}), "
                       f"m={P['m']}, t={t}, L={P['L']}, K={P['K']}, delta={P['delta']}, g={P['g']}; "
                       f"numpy oracle port of run_pipeline, {sec:.2f} s per run"), sec


# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            # one GPU, or the node's first `world` GPUs (local rank r drives GPU r; idle GPUs
            # of a larger box would drag the median down)
            ids = [f"--id={self.idx}"] if isinstance(self.idx, int) else [f"--id={','.join(map(str, self.idx))}"]
            self.proc = subprocess.Popen(["nvidia-smi", *ids, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            ref, sec = cpu_reference(args.cpu_sample, args.steps, min(args.warmup, 1))
            line = dict(metric=METRIC, value=ref["value"], unit="points/s", n_gpus=args.gpus, steps=args.steps,
                        warmup=args.warmup, ms_per_step=sec * 1e3, higher_is_better=True, scaling="strong",
                        vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
                        config=dict(workload="geek-dense-sift-like (CPU sample)", n=args.cpu_sample,
                                    **PARAMS),
                        cpu_baseline=ref, e2e=dict(value=ref["value"], unit="points/s", h2d_bytes_per_step=0,
                                                   d2h_bytes_per_step=0))
            print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_10515_b200 as G
    from paper_2106_10515_b200 import _lib
    from paper_2106_10515_b200.engine import split_data
    from paper_2106_10515_b200.synth import gaussian_mixture_device

    P = PARAMS
    n = args.n
    t = n // P["points_per_bucket"]
    lo, hi = split_data(n, world)[rank]
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(P["g"]),
                           homo=G.HomoTransformParams(P["m"], t, seed=P["tseed"]),
                           seeding=G.SeedingParams(P["K"], P["L"], min_group_size=P["delta"], seed=P["sseed"]))
    X = gaussian_mixture_device(n, P["d"], P["clusters"], P["separation"], P["data_seed"], lo, hi - lo)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(Xs):
        return G.run_pipeline_shard(Xs, n, cfg)

    def max_over_ranks(v):
        if world == 1:
            return v
        tt = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    out = None
    for _ in range(args.warmup):
        out = step(X)
    barrier()
    # ---- timed region: resident data --------------------------------------
    # one sampler for the job: rank 0 polls every GPU of the node (an
    # nvidia-smi per rank perturbs the timed steps)
    clocks = ClockSampler(local if world == 1 else list(range(int(os.environ.get("LOCAL_WORLD_SIZE", world)))))
    if rank == 0:
        clocks.start()
    timer = _lib.CallTimer()
    _lib.set_call_timer(timer)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        out = step(X)
    e1.record()
    barrier()
    _lib.set_call_timer(None)
    my_ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(my_ms * args.steps) / args.steps
    rank_ms = [my_ms]
    if world > 1:
        allt = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(world)]
        dist.all_gather(allt, torch.tensor([my_ms], dtype=torch.float64, device="cuda"))
        rank_ms = [round(float(x.item()), 3) for x in allt]
    clk = clocks.stop()
    calls = timer.ms_by_name()
    info = dict(out.info)
    stage = {k: round(v, 4) for k, v in out.timings.items()}  # CUDA-event stage times of the last step
    k_star, ngroups = out.k_star, len(out.seed_groups) if n <= 10**6 else out._groups.count

    # ---- launches per step (torch profiler / CUPTI, untimed) ------------------
    launches = None
    try:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(X)
            torch.cuda.synchronize()
        launches = sum(1 for e in prof.events() if e.device_type.name == "CUDA" and "geek::" in e.name)
        if os.environ.get("GEEK_PROFILE") and rank == 0:
            print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=45), file=sys.stderr)
        if os.environ.get("GEEK_TRACE"):  # CPU + GPU timeline of one step (all ranks step; rank 0 exports)
            with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as tr:
                step(X)
                torch.cuda.synchronize()
            if rank == 0:
                tr.export_chrome_trace(os.environ["GEEK_TRACE"])
    except Exception as exc:  # profiler unavailable: leave null
        print(f"[bench] launch count unavailable: {exc}", file=sys.stderr)

    # ---- e2e: pinned host -> device -> pipeline -> labels back ---------------
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
        Xh.copy_(X)
        del X, out
        torch.cuda.empty_cache()
        lab_h = torch.empty(hi - lo, dtype=torch.int64, pin_memory=True)
        step(Xh)  # warm the engine's device row buffer
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            # the public API on pinned host rows: the engine copies them to the
            # GPU in chunks (each projected as it lands), the labels come back
            o = step(Xh)
            lab_h.copy_(o.labels_device, non_blocking=True)  # labels device -> host, pinned
        f1.record()
        barrier()
        e2e_ms = max_over_ranks(f0.elapsed_time(f1)) / args.steps
        e2e = dict(value=n / (e2e_ms / 1e3), unit="points/s", h2d_bytes_per_step=int(Xh.numel() * 4) * world,
                   d2h_bytes_per_step=int(lab_h.numel() * 8) * world, ms_per_step=round(e2e_ms, 3))

    # ---- roofline of the dominant kernel -------------------------------------
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    roof = None
    dom = None
    if info.get("screen_ms"):
        # tcgen05 screen: algorithmic work = the n x k x d distance GEMM
        sec = info["screen_ms"] / 1e3
        kk = info.get("centers", ngroups)
        flops = 2.0 * (hi - lo) * kk * P["d"]
        mode = info.get("screen_mode", 16)
        f16 = mode == 16
        tile_n = 192
        nct = -(-kk // tile_n)
        kexec = tile_n * (nct - 1) + -(-(kk - tile_n * (nct - 1)) // 16) * 16  # last tile at N = valid rounded to 16
        nl = hi - lo
        # 3 products (hi*hi, hi*lo, lo*hi) + the |c'|^2 K slice (16 f16 / 8 tf32 wide)
        exec_flops = 2.0 * nl * kexec * ((3 if mode != 1 else 1) * P["d"] + (16 if f16 else 8))
        exec_peak = peaks.get("bf16_tflops", 1590.0) if f16 else 1066.0
        roof = dict(kernel="tc_screen_kernel", bound="tensor", achieved=flops / sec / 1e12, unit="TFLOP/s",
                    peak=peaks.get("bf16_tflops", 1590.0),
                    # dram read + write per launch from `ncu --set full` (profiles/r1_kernels.md: 51.23 GB
                    # + 8.00 GB at n = 1e8), scaled to this rank's points; = the algorithmic X + top-list + |x'|^2 bytes
                    traffic=59.23e9 * nl / 1e8,
                    peak_source="MEASURED_PEAKS.json bf16_tflops (dense bf16 cuBLAS; the kind::f16 screen runs on "
                                "the same tensor rate; kind::tf32 runs at 1066 TFLOP/s, tools/tc_rate.cu)",
                    screen=("FP16x3" if f16 else "TF32x3" if mode == 3 else "TF32"),
                    executed_tflops=exec_flops / sec / 1e12,
                    executed_frac_of_peak=exec_flops / sec / 1e12 / exec_peak,
                    kernel_ms=info["screen_ms"],
                    note=f"achieved = algorithmic flops 2*n*k*d (k={kk}, d={P['d']}) per launch / CUDA-event time; "
                         f"the kernel executes 3 products (hi*hi, hi*lo, lo*hi) of "
                         f"{'f16 parts of power-of-two scaled' if f16 else 'TF32 parts of'} operands over k padded "
                         f"to {kexec} plus the |c'|^2 K-slice, for exact float64 labels after the recheck")
        roof["frac"] = roof["achieved"] / roof["peak"]
    elif "geek_project_keys" in calls:
        dom = "geek_project_keys"
    if dom == "geek_project_keys":
        per = calls[dom][0] / calls[dom][1] / 1e3
        nl = hi - lo
        byts = nl * (4 * P["d"] + 8 * P["m"])
        roof = dict(kernel="project_kernel", bound="hbm", achieved=byts / per / 1e9, unit="GB/s",
                    peak=peaks.get("hbm_gbs", 6650.0), traffic=None,
                    note="algorithmic bytes = n*(4d read + 8m key write) per launch")
        roof["frac"] = roof["achieved"] / roof["peak"]
    elif dom == "geek_assign_l2":
        per = calls[dom][0] / calls[dom][1] / 1e3
        nl = hi - lo
        byts = nl * (4 * P["d"] + 16)
        roof = dict(kernel="assign_l2_kernel", bound="hbm", achieved=byts / per / 1e9, unit="GB/s",
                    peak=peaks.get("hbm_gbs", 6650.0), traffic=None,
                    note=f"exact float64 brute force over k={ngroups} centers; algorithmic bytes n*(4d+16)")
        roof["frac"] = roof["achieved"] / roof["peak"]

    if rank == 0:
        cpu, _ = cpu_reference(args.cpu_sample, 1, 0)
        line = dict(metric=METRIC, value=n / (ms / 1e3), unit="points/s", n_gpus=world, steps=args.steps,
                    warmup=args.warmup, ms_per_step=round(ms, 3), higher_is_better=True, scaling="strong",
                    vs_baseline=None, dtype="f64", data="synthetic",
                    config=dict(workload="geek-dense-sift-like 100M x 128 (BASELINE configs[1])" if n == 100_000_000
                                else f"geek-dense-sift-like {n} x 128", n=n, t=t, **PARAMS,
                                parallelism=f"points-sharded x{world} (g_logical={P['g']})",
                                l2="inputs 51 GB >> 126 MB L2; no flush needed"),
                    e2e=e2e, gpu_launches=(launches * args.steps if launches is not None else None),
                    clocks=clk, roofline=roof, cpu_baseline=cpu,
                    stages_s=stage, rank_ms_per_step=rank_ms, k_star=k_star, seed_groups=ngroups,
                    calls_ms={k: round(v[0] / v[1], 3) for k, v in sorted(calls.items(), key=lambda kv: -kv[1][0])},
                    info=info)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
