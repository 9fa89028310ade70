#!/usr/bin/env python
"""Headline benchmark: rank-pair 1D convolutions/s of the canonical Hartree
convolution (BASELINE.json metric) on config 2 — n = 16385, R_f = 500 density
terms, R_N = 41 Newton-kernel terms (M = 20), 3 x 500 x 41 = 61,500 windowed
FP64 convolutions of length 16385 per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N > 1).  The path partitions by rank pair
with no data-path collective (output factors stay on their devices), so by
default every rank convolves its own R_f = 500 density columns (a rank-specific
shard of an N x 500-column seeded density): weak scaling, per-GPU work fixed.
`--strong` instead shards the fixed 500 columns of config 2 across the ranks
(the north star's 20,500 rank pairs split over 1/2/4/8 GPUs).  Rank 0 prints ONE
JSON line.  The timed region is bracketed by a barrier and
torch.cuda.synchronize() on both sides, timed with CUDA events on the libtgb
context stream, max over ranks.

`--impl reference` times the reference's own CPU code for the path
(oracle/_ref: proj/src/fft.cpp + tensor.cpp compiled from /root/reference),
or the oracle restatement if that library is absent, on a bounded sample of
the same workload with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

CFG = 2
N_GRID = 16385
R_F = 500
METRIC = "rank-pair 1D convolutions/s (canonical Hartree conv)"
UNIT = "convs/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


FP64_TFLOPS = 36.6  # DFMA microbenchmark on this pool's B200 (profiles/r01_box_probe.txt)


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU reference arm

def cpu_reference_sample(budget_s: float = 12.0, threads: int | None = None) -> dict:
    """Time the reference's conv_central_many (proj/src/fft.cpp:97-122, the
    per-column kernel of tg::convolve) on a bounded sample of the config-2
    workload: one axis, `cols` density columns against kernel columns in
    turn, all host threads.  Returns units/s (one unit = one windowed length-n
    convolution, as in the GPU metric)."""
    import ctypes as C

    from oracle import oracle as O
    from paper_1504_06289_b200.inputs import hartree_case

    threads = threads or os.cpu_count() or 1
    case = hartree_case(CFG, nsamples=1)
    U = np.asfortranarray(case.theta.factor[0])
    K = case.kernel.tensor.factor[0]
    R = O.rlib()
    kind = "reference" if R is not None else "port"
    n = N_GRID
    cols = min(R_F, max(threads, 16))
    out = np.zeros((n, cols), order="F")
    Usub = np.asfortranarray(U[:, :cols])

    def run_one(j):
        v = np.ascontiguousarray(K[:, j])
        if R is not None:
            rc = R.ref_conv_central_many(C.c_longlong(n), C.c_longlong(cols), C.c_void_p(Usub.ctypes.data),
                                         C.c_void_p(v.ctypes.data), C.c_void_p(out.ctypes.data), C.c_int(threads))
            if rc:
                raise RuntimeError(R.ref_last_error().decode())
        else:
            out[:] = O.conv_central_many(Usub, v)

    t0 = time.perf_counter()
    units = 0
    j = 0
    while True:
        run_one(j % K.shape[1])
        units += cols
        j += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return {"value": units / el, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"axis 0 of config 2: {cols} density columns x {j} kernel columns "
                      f"(n={n}, reference radix-2 FFT length 65536), {units} convolutions in {el:.1f} s"}


def run_reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    results = []
    for _ in range(args.warmup):
        cpu_reference_sample(budget_s=1.0)
    for _ in range(args.steps):
        results.append(cpu_reference_sample(budget_s=max(2.0, 60.0 / max(args.steps, 1))))
    vals = [r["value"] for r in results]
    v = statistics.median(vals)
    base = dict(results[-1])
    base["value"] = v
    per_step_ms = 1000.0 * (3 * R_F * 41) / v
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config 2: Hartree convolution n=16385, R_f=500, R_N=41 (M=20)", "n": N_GRID,
                   "R_f": R_F, "R_N": 41, "parallelism": "host threads", "steps_are": "bounded samples"},
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--strong", action="store_true", help="shard config 2's fixed 500 density columns")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    import paper_1504_06289_b200 as tg
    from paper_1504_06289_b200.inputs import hartree_case

    strong = args.strong or world == 1
    total_f = R_F if strong else R_F * world
    case = hartree_case(CFG, rank=total_f, nsamples=10_000)
    # shard the density columns (rank pairs i + R_f j with i in this rank's block)
    lo = rank * total_f // world
    hi = (rank + 1) * total_f // world
    theta = tg.CanonicalTensor3([f[:, lo:hi] for f in case.theta.factor], case.theta.weight[lo:hi])
    kern = case.kernel.tensor
    ra, rb = theta.rank(), kern.rank()
    n = N_GRID
    units_local = 3 * ra * rb
    units_total = 3 * total_f * rb

    stream = torch.cuda.Stream(device=dev)
    ctx = tg.Context(local, stream=stream.cuda_stream)
    d_theta = tg.DeviceCP.from_host(theta, device=dev)
    d_kern = tg.DeviceCP.from_host(kern, device=dev)
    d_out = tg.DeviceCP.empty([n, n, n], ra * rb, device=dev)
    h = case.grid.h

    def step():
        tg.hartree_potential(d_theta, d_kern, h, ctx, out=d_out)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs)
    ctx.set_profiling(True)
    ctx.profile_read()
    ctx.reset_launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1)
    launches = ctx.launch_count()
    pair_ms, pair_launches = ctx.profile_read()
    ctx.set_profiling(False)

    ms_t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total = float(ms_t.item())
    ms_step = ms_total / args.steps
    value = units_total / (ms_step / 1e3)

    # ---- validation outside the timed region: V_H at 10^4 sample points, one
    # NCCL allreduce of the per-rank partial sums (the path's only exchange).
    pts = torch.as_tensor(case.samples, device=dev)
    part = tg.value_at_points(d_out, pts, ctx)
    wt = d_out.weight  # weights already in place
    torch.cuda.synchronize()
    if world > 1:
        dist.all_reduce(part)
    samples_vh = part.cpu().numpy()

    # ---- roofline of the dominant kernel (pair convolution kernel, one launch = one axis)
    hbm_peak, peak_kind = peaks()
    nd = 21  # distinct kernel columns (M + 1)
    bytes_launch = 8.0 * n * ra * rb + 8.0 * n * (ra + rb)
    # each axis launches the pair kernel once per spectrum form (real / complex);
    # the form that disagrees with the device-side symmetry flag exits at once,
    # so the working launches are 3 per step (its ~4 us is kept in pair_ms)
    work_launches = 3 * args.steps
    avg_launch_ms = pair_ms / max(min(pair_launches, work_launches), 1)
    achieved = bytes_launch / (avg_launch_ms / 1e3) / 1e9
    traffic = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        try:
            traffic = json.loads(tj.read_text()).get("pair_kernel_dram_bytes_per_launch")
        except Exception:
            traffic = None
    # FP64 work actually issued per launch (inverse FFT length m = 2N = 25600)
    m = 25600
    N = m // 2
    flops_pair = 5.0 * N * np.log2(N) + 16.0 * N  # complex FFT + split + product (nominal)
    fp64_tflops = ra * nd * flops_pair / (avg_launch_ms / 1e3) / 1e12

    # ---- e2e through the C-ABI with pinned HOST buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        th = tg.CanonicalTensor3([torch.empty((ra, n), dtype=torch.float64).pin_memory().numpy().T for _ in range(3)],
                                 theta.weight)
        for ax in range(3):
            th.factor[ax][:] = theta.factor[ax]
        kh = tg.CanonicalTensor3([torch.empty((rb, n), dtype=torch.float64).pin_memory().numpy().T for _ in range(3)],
                                 kern.weight)
        for ax in range(3):
            kh.factor[ax][:] = kern.factor[ax]
        oh = tg.CanonicalTensor3([torch.empty((ra * rb, n), dtype=torch.float64).pin_memory().numpy().T
                                  for _ in range(3)], np.zeros(ra * rb))
        h2d = sum(f.nbytes for f in th.factor) + sum(f.nbytes for f in kh.factor)
        d2h = sum(f.nbytes for f in oh.factor)
        tg.hartree_potential(th, kh, h, ctx, out=oh)  # warm (staging buffers)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            tg.hartree_potential(th, kh, h, ctx, out=oh)
        el = time.perf_counter() - t0
        el_t = torch.tensor([el], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(el_t, op=dist.ReduceOp.MAX)
        e2e_step = float(el_t.item()) / args.e2e_steps
        e2e = {"value": units_total / e2e_step, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_step * 1e3, "steps": args.e2e_steps,
               "timing": "host wall clock around the C-ABI call (includes pinned H2D + D2H), max over ranks"}
        del oh

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(budget_s=12.0)
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "unavailable", "sample": str(exc)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config 2: Hartree convolution (tg::hartree_potential) n=16385, R_f=500, "
                               "R_N=41 (M=20), 61,500 windowed FP64 1D convolutions per step",
                   "n": n, "R_f": R_F, "R_N": rb, "units_per_step": units_total,
                   "parallelism": (f"dp{world} (config 2's {R_F} density columns sharded)" if strong else
                                   f"dp{world} ({R_F} density columns per GPU, rank-specific shards)"),
                   "l2": "no flush needed: each step writes 8.06 GB of factors (> 126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "pair_kernel (inverse FFT + window + store, one launch per axis)",
                     "bytes_per_launch": bytes_launch, "avg_launch_ms": avg_launch_ms,
                     "launch_share_of_step": pair_ms / ms_local if ms_local else None,
                     "fp64": {"achieved_tflops_nominal": fp64_tflops, "peak_tflops": FP64_TFLOPS,
                              "frac": fp64_tflops / FP64_TFLOPS,
                              "note": "nominal 5 N log2 N + 16 N flops per inverse transform, N = 12800"}},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "validation": {"sample_points": int(len(samples_vh)), "vh_sample_checksum": float(np.sum(samples_vh)),
                       "allreduce": "nccl" if world > 1 else "none (single rank)"},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
