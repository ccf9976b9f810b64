"""Benchmark: grid-point updates per second of the acoustic time loop behind
Operator.apply on BASELINE.json config 2 (so=8, 512^3 interior + 40-point
damping = 592^3, 512x512 receivers, nt=500), one B200 per rank.

A *step* is one full ``apply`` time loop (nt time steps) over device-resident
buffers. ``value`` = all ranks' points*nt per step / max-over-ranks device
time; ``e2e`` = the same metric through the public ``Operator.apply`` with
host numpy buffers (H2D + D2H inside the timed region).

    python bench.py [--gpus N --steps K --warmup W --so 8 --impl ours|reference]

Multi-GPU (torchrun, N>1): every rank runs its own config-2 problem (weak
scaling, no data-path collective); the result is max-reduced over ranks.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# SURVEY.md §8d algorithmic accounting (f32, every point counted once/step)
BYTES_PER_PT = {"acoustic": 20,   # read u[t], u[t-1], m, damp; write u[t+1]
                "tti": 48}        # read p,p-,r,r-,m,damp,eps,delta,th,ph; write p+,r+
FLOPS_PER_PT = {"acoustic": lambda so: 4.5 * so + 11,
                "tti": lambda so: 13.5 * so + 39}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index),
                     "--query-gpu=" + self.Q, "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows else None,
                "reasons": reasons, "samples": len(self.rows)}


def _reference_module():
    """The unmodified reference (stencilc) from baseline/_ref (offline
    install that travels to the GPU box), else None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "stencilc")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import stencilc.symbolic as RS
        from stencilc.backend.operator import Operator as RefOp
    except Exception:
        return None
    return RS, RefOp


def _ref_apply(RefOp, eqs, fill, steps, dt, workers):
    """Reference Operator.apply on seeded inputs: one warm-up step, then
    ``steps`` timed; returns seconds per step of the time-loop section."""
    op = RefOp(eqs, mode="advanced", dtype="f32")
    bufs = op.allocate(steps + 1)
    fill(bufs)
    op.apply(steps=1, buffers=bufs, dt=dt, workers=workers)
    t0 = time.perf_counter()
    _, rep = op.apply(steps=steps + 1, buffers=bufs, dt=dt, workers=workers,
                      t_m=1, t_M=steps)
    wall = time.perf_counter() - t0
    loop = max(rep.values(), key=lambda v: v["time"])["time"]
    return min(loop, wall) / steps


def cpu_sample(so: int, steps: int = 2, x_planes: int = 64, kind="acoustic",
               npts_full: int = 592 ** 3, nrec_full: int = 512 * 512):
    """CPU baseline: the REFERENCE's own Operator.apply
    (stencilc from baseline/_ref, advanced mode, f32) on bounded samples of
    the config-2 workload, extrapolated linearly to the full problem:

    * stencil: an x-slab of ``x_planes`` x 592 x 592 (damping included) with
      all host threads (the reference chunks x across ``workers``);
    * receivers and the source: 1024 receivers + the source on a small grid
      with one worker (the reference's per-point loop is GIL-bound; more
      workers are slower), scaled linearly to 262,144;
    * per step: stencil time x (592^3 / slab points) + receiver time x 256.

    Falls back to the oracle port (numpy restatement, vectorised sparse
    loops, kind "port") when the reference is not installed. TTI: the
    reference's advanced-mode compile takes 5-16 min at so >= 12 (SURVEY
    §0.1 #2), so the TTI sample is the port on a 48^3 so=4 operator."""
    import oracle
    import workloads
    ref = _reference_module() if kind == "acoustic" else None
    if kind == "tti":
        from paper_1807_03032_b200.backend.operator import Operator
        o2, _, _, _ = workloads.config3(so=4, n=32, nbl=8, nt=steps)
        op = Operator(o2.eqs, mode="advanced", dtype="f32", fuse=False)
        _, bufs, dt, meta = workloads.config3(so=4, n=32, nbl=8, nt=steps)
        bufs = {k: v for k, v in bufs.items()}
        workers = os.cpu_count() or 1
        t0 = time.perf_counter()
        oracle.apply(op, steps, bufs, workers=workers, dt=dt)
        sec = time.perf_counter() - t0
        npts = int(np.prod(meta["shape"])) * steps
        return npts / sec / 1e9, workers, sec, \
            "TTI so=4 %s, %d time steps (oracle DSE excluded), numpy %s" % (
                "x".join(map(str, meta["shape"])), steps, np.__version__), \
            "port"
    if ref is None:
        op, bufs, dt, meta = workloads.config2(so=so, nt=steps,
                                               x_planes=x_planes + 32,
                                               nrec_side=64)
        workers = os.cpu_count() or 1
        t0 = time.perf_counter()
        oracle.apply(op, steps, bufs, workers=workers, dt=dt)
        sec = time.perf_counter() - t0
        npts = int(np.prod(meta["shape"])) * steps
        return npts / sec / 1e9, workers, sec, \
            "oracle port (reference not installed): config-2 x-slab %s, " \
            "so=%d, %d steps, %d receivers, numpy %s" % (
                "x".join(map(str, meta["shape"])), so, steps, meta["nrec"],
                np.__version__), "port"
    RS, RefOp = ref
    workers = os.cpu_count() or 1
    full = {"nrec": nrec_full}
    # stencil: x-slab, no sparse statements
    _, sb, dt, sm = workloads.config2(so=so, nt=steps + 1, x_planes=x_planes,
                                      nrec_side=1)
    eqs = workloads.acoustic_equations(sm["shape"], sm["h"], so,
                                       sm["src_coords"], [], S=RS)[:1]

    def fill_slab(b):
        for k in ("m", "damp"):
            b[k].data[...] = sb[k].data
        H = so // 2
        rng = np.random.default_rng(1)
        inner = b["u"].data[0:2, H:-H, H:-H, H:-H]
        inner[...] = rng.uniform(-1, 1, inner.shape).astype(np.float32)
    w0 = time.perf_counter()
    t_sten = _ref_apply(RefOp, eqs, fill_slab, steps, dt, workers)
    slab_pts = int(np.prod(sm["shape"]))
    # sparse: the source + 1024 receivers on a 64^3 model (per-point cost
    # scaled linearly; config 4 has no receivers: its sources are negligible)
    nrec = 1024
    _, rb, _, rm_ = workloads.config2(so=so, n=48, nbl=8, nt=steps + 1,
                                      nrec_side=32)
    eqs2 = workloads.acoustic_equations(rm_["shape"], rm_["h"], so,
                                        rm_["src_coords"], rm_["rec_coords"],
                                        S=RS)
    eqs_sp = eqs2[1:]                       # injection + interpolation only

    def fill_sp(b):
        for k in ("m", "src"):
            if k in b:
                b[k].data[...] = rb[k].data[:b[k].data.shape[0]]
    t_sp = _ref_apply(RefOp, eqs_sp, fill_sp, steps, dt, 1)
    per_step = t_sten * npts_full / slab_pts + t_sp * full["nrec"] / nrec
    sec = time.perf_counter() - w0            # wall time of this sample
    return npts_full / per_step / 1e9, workers, sec, \
        ("reference stencilc (baseline/_ref) Operator.apply, advanced, f32, "
         "numpy %s: stencil timed on a %s x-slab with %d workers (%.3f s/step "
         "-> %.2f s/step at 592^3), source + %d receivers with 1 worker "
         "(%.3f s/step -> %.2f s/step for %d receivers); extrapolated "
         "linearly to %.1f s per time step of %d points, %d timed steps each"
         % (np.__version__, "x".join(map(str, sm["shape"])), workers, t_sten,
            t_sten * npts_full / slab_pts, nrec, t_sp,
            t_sp * full["nrec"] / nrec, full["nrec"], per_step, npts_full,
            steps)), "reference"


def workload_label(args, shape):
    """The `config.workload` string of the default single-domain workloads;
    the reference arm reports the same one (its step is a bounded sample)."""
    dims = "x".join(map(str, shape))
    if args.workload == "config4":
        return ("config4: 3D acoustic so=%d, 1024^3 interior per GPU "
                "(global %s), nt=%d, weak scaling, one source per slab"
                % (args.so, dims, args.nt if args.nt != 500 else 200))
    if args.workload == "config1":
        return ("config1: 3D acoustic so=%d, 128^3 interior + 10 damping (%s), "
                "h=10 m, nt=%d, 101 receivers" % (args.so, dims, args.nt))
    if args.op == "acoustic":
        return ("config2: 3D acoustic so=%d, %d^3 interior + 40 damping (%s), "
                "h=20 m, nt=%d, 512x512 receivers"
                % (args.so, args.n, dims, args.nt))
    return ("config3: 3D TTI p/r so=%d, %d^3 interior + 40 damping (%s), "
            "h=20 m, nt=%d, no receivers" % (args.so, args.n, dims, args.nt))


def reference_arm(args, rank):
    if rank != 0:
        return 0
    full = {"npts_full": 592 ** 3, "nrec_full": 512 * 512}
    if args.workload == "config4":
        # weak scaling: 1024^3 interior per GPU, no receivers, no damping
        # (the zero damp field is still read, as on the GPU)
        full = {"npts_full": args.gpus * 1024 ** 3, "nrec_full": 0}
    elif args.workload == "config1":
        full = {"npts_full": 148 ** 3, "nrec_full": 101}
    for _ in range(args.warmup):
        cpu_sample(args.so, steps=1, x_planes=16, kind=args.op, **full)
    vals, secs = [], []
    workers = 1
    sample = ""
    kind = "port"
    for _ in range(args.steps):
        v, workers, sec, sample, kind = cpu_sample(args.so, kind=args.op,
                                                   **full)
        vals.append(v)
        secs.append(sec)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": "GPts/s", "value": value,
            "unit": "GPts/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_label(
                           args, (148,) * 3 if args.workload == "config1"
                           else (1024 * args.gpus, 1024, 1024)
                           if args.workload == "config4"
                           else (args.n + 80,) * 3),
                       "operator": args.op, "so": args.so,
                       "step": "bounded CPU sample of the same per-point "
                               "work: " + sample},
            "cpu_baseline": {"value": value, "unit": "GPts/s",
                             "cores": workers, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": "GPts/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def fp32_peak() -> float:
    """Nominal dense FP32 TFLOP/s of this GPU: SMs x 128 FP32 lanes x 2 flop
    (FMA) x max SM clock."""
    import torch
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    _, _, peaks = measured_peaks()
    mhz = peaks.get("sm_max_mhz", 1965.0)
    return props.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12


def ncu_traffic(op: str, so: int):
    """DRAM bytes (read + write) per launch of the dominant kernel(s) from
    the committed ncu --set full capture (profiles/traffic.json), for the
    op/space order that capture was taken at; None otherwise."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "profiles", "traffic.json")
    try:
        with open(path) as f:
            ks = json.load(f)["kernels"].get(op, {})
    except (OSError, ValueError):
        return None
    tag = "<float, %d," % so if op == "acoustic" else "<%d>" % so
    hits = [v for k, v in ks.items() if tag in k]
    if not hits:
        return None
    return sum(v["dram_read_bytes"] + v["dram_write_bytes"] for v in hits)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--so", type=int, default=None)
    ap.add_argument("--op", default="acoustic", choices=("acoustic", "tti"))
    ap.add_argument("--nt", type=int, default=500)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--nrec-side", type=int, default=512)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--tti-nt", type=int, default=100,
                    help="time steps of the config-3 TTI sub-record of the "
                         "default acoustic run (0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--slabs", action="store_true",
                    help="x-slab decomposed path even on one GPU")
    ap.add_argument("--workload", default=None,
                    choices=("config1", "config2", "config4", "config5"),
                    help="config4: BASELINE config 4 (1024^3 interior per "
                         "GPU, so=8, nt=200) through the slab path at any N")
    ap.add_argument("--no-overlap", action="store_true",
                    help="multi-GPU: exchange ghost planes after the whole "
                         "step instead of overlapping it with the interior")
    args = ap.parse_args()
    if args.so is None:
        args.so = 8 if args.op == "acoustic" else 12

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload is None:
        # N > 1: BASELINE config 4 (weak scaling, 1024^3 interior per GPU);
        # config 5 (TTI strong scaling) via --workload config5
        args.workload = "config4" if world > 1 and args.op == "acoustic" \
            else "config2"
    if args.impl == "reference":
        return reference_arm(args, rank)

    import torch
    import torch.distributed as dist
    import workloads
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if world > 1 or args.slabs or args.workload in ("config4", "config5"):
        return run_slabs(args, world, rank, local)
    if args.op == "acoustic" and args.workload == "config1":
        args.so = 4
        if args.nt == 500:
            args.nt = 200                # config 1's own nt
        op, bufs, dt, meta = workloads.config1(nt=args.nt)
    elif args.op == "acoustic":
        op, bufs, dt, meta = workloads.config2(so=args.so, n=args.n, nt=args.nt,
                                               nrec_side=args.nrec_side)
    else:
        op, bufs, dt, meta = workloads.config3(so=args.so, n=args.n, nt=args.nt)
    npts = int(np.prod(meta["shape"]))
    run = op.prepare(args.nt, bufs, dt=dt)
    for _ in range(args.warmup):
        run.run(profile=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # a working set that fits the 126 MB L2 (config 1: 70 MB) is flushed
    # between timed iterations by writing a 256 MB buffer, outside the events
    small = meta.get("l2_resident", False)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda") \
        if small else None
    barrier()
    with ClockSampler(local) as clk:
        if small:
            ms = 0.0
            for _ in range(args.steps):
                flush.fill_(1.0)
                e0.record()
                run.run(profile=False)
                e1.record()
                e1.synchronize()
                ms += e0.elapsed_time(e1)
        else:
            e0.record()
            for _ in range(args.steps):
                run.run(profile=False)
            e1.record()
        barrier()
    if not small:
        ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # per-stage CUDA-event times for the roofline: one profiled pass right
    # after the timed region (same power/clock state as the timed loop)
    rep = run.run(profile=True)
    sec = [v for v in rep.values() if "stages" in v][0]
    if not sec["fast_path"]:
        raise SystemExit("fused kernel not selected")
    stages = sec["stages"]
    dense_s = [v for k, v in stages.items() if k.startswith("dense")][0]
    kern_ms = dense_s * 1e3 / args.nt
    launches = run.plan.launches * args.steps
    loop_ms = run.plan.total_ms
    value = world * npts * args.nt * args.steps / (ms / 1e3) / 1e9

    # end to end through the public API with host buffers: the device-resident
    # run is released first; one untimed warm-up apply (allocator and pinned
    # staging pools), then e2e_steps timed ones (H2D + loop + D2H each)
    h2d = d2h = 0
    run.close()
    del run
    gc.collect()
    torch.cuda.empty_cache()
    e2e_n = max(args.e2e_steps, 0)

    from paper_1807_03032_b200.backend import operator as opmod

    def e2e_apply():
        # the public call: Operator.apply on the caller's pinned host buffers
        # (H2D of every input, the time loop, D2H of every written function);
        # the prepared run (plan, programs, CUDA graph) is reused across
        # applies of the same problem, as a user's shot loop would
        op.apply(args.nt, bufs, dt=dt)
        r = opmod._RUN_CACHE["run"]
        return r.h2d_bytes, r.d2h_bytes

    first_s = None
    if e2e_n:
        t0 = time.perf_counter()
        e2e_apply()
        first_s = time.perf_counter() - t0
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_n):
        h2d, d2h = e2e_apply()
    barrier()
    e2e_s = (time.perf_counter() - t0) / max(e2e_n, 1)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = world * npts * args.nt / e2e_s / 1e9 if e2e_n else None
    op.release()

    peak, peak_kind, peaks = measured_peaks()
    from paper_1807_03032_b200.backend.runtime import measure_fp32_tflops
    fp32_measured = measure_fp32_tflops()   # after the timed region
    bpp = BYTES_PER_PT[args.op]
    achieved = bpp * npts / (kern_ms / 1e3) / 1e9
    flops = FLOPS_PER_PT[args.op](args.so)
    line = {
        "metric": "GPts/s", "value": value, "unit": "GPts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded two-layer velocity, damping layer, 10 Hz "
                "Ricker at the centre, 101 receivers)"
        if args.workload == "config1" else
        ("synthetic (seeded 8-layer velocity, damping layer, Ricker "
                 "source, %d receivers)" % meta["nrec"]) if args.op == "acoustic"
        else "synthetic (seeded two-layer velocity, Gaussian-smoothed eps/delta/"
             "theta/phi, damping layer, Ricker source into p and r)",
        "config": {"workload": workload_label(args, meta["shape"]),
                   "operator": args.op,
                   "so": args.so, "grid": list(meta["shape"]), "nt": args.nt,
                   "step": "one Operator.apply time loop (nt time steps)",
                   "l2": ("flushed between timed iterations (256 MB write): "
                          "the working set fits the 126 MB L2 within a run"
                          if meta.get("l2_resident") else
                          "no flush: the wavefields (>= 2.6 GB) exceed the 126 "
                          "MB L2 every time step"),
                   "parallelism": "replica per GPU" if world > 1 else "1 GPU"},
        "gflops": value * flops,
        # the FP32 roofline next to the HBM one: minimal
        # closed-form flops/pt x points / kernel time vs the nominal FP32
        # peak (148 SMs x 128 lanes x 2 flop x max SM clock)
        "roofline_fp32": {"bound": "fp32", "unit": "TFLOP/s",
                          "flops_per_pt": flops,
                          "achieved": flops * npts / (kern_ms / 1e3) / 1e12,
                          "peak": fp32_peak(),
                          "peak_kind": "nominal (148 SMs x 128 lanes x 2 x "
                                       "max SM clock)",
                          "peak_measured": fp32_measured,
                          "frac": flops * npts / (kern_ms / 1e3) / 1e12
                          / fp32_peak()},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.op, args.so),
                     "traffic_unit": "bytes/launch (ncu dram read+write, "
                                     "profiles/traffic.json)",
                     "kernel": "%s so=%d (%.3f ms/launch, %d B/pt x %d pts)"
                               % ("acoustic_kernel" if args.op == "acoustic"
                                  else ("tti_inner+tti_outer"
                                        if os.environ.get("SC_TTI_PLAIN")
                                        else "tti_g1z_tma+tti_upd1z_tma"),
                                  args.so, kern_ms,
                                  bpp, npts),
                     "peak_kind": peak_kind},
        "e2e": {"value": e2e, "unit": "GPts/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "s_per_apply": e2e_s if e2e_n else None,
                "first_apply_s": first_s,
                "note": "Operator.apply on pinned host buffers; the first "
                        "apply prepares (tables, programs, graph capture) "
                        "and is untimed, later applies reuse the prepared "
                        "run"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "stage_ms_per_step": {k: v * 1e3 / args.nt for k, v in stages.items()},
        "timestep_ms": loop_ms / args.nt,
    }
    if args.op == "acoustic" and args.workload == "config2" and \
            args.tti_nt > 0:
        # driver-timed TTI next to the headline: config 3 (so=12, 592^3) over
        # a short horizon, after this run's buffers are released
        del bufs
        gc.collect()
        torch.cuda.empty_cache()
        line["tti"] = tti_subrecord(args, barrier)
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, sec_cpu, sample, kind = cpu_sample(args.so, kind=args.op)
        line["cpu_baseline"] = {"value": v, "unit": "GPts/s", "cores": cores,
                                "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def tti_subrecord(args, barrier):
    """BASELINE config 3 (TTI p/r, so=12, 512^3 + 40 damping = 592^3) timed
    like the headline (device-resident, CUDA events around ``steps`` applies
    of ``tti_nt`` time steps, clocks sampled), with the pass times of one
    profiled apply right after for the 48 B/pt roofline."""
    import torch
    import workloads
    so, nt = 12, args.tti_nt
    op, bufs, dt, meta = workloads.config3(so=so, n=args.n, nt=nt)
    npts = int(np.prod(meta["shape"]))
    run = op.prepare(nt, bufs, dt=dt)
    for _ in range(max(args.warmup, 2)):
        run.run(profile=False)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        e0.record()
        for _ in range(args.steps):
            run.run(profile=False)
        e1.record()
        barrier()
    ms = e0.elapsed_time(e1)
    rep = run.run(profile=True)
    sec = [v for v in rep.values() if "stages" in v][0]
    dense_s = [v for k, v in sec["stages"].items() if k.startswith("dense")][0]
    kern_ms = dense_s * 1e3 / nt
    launches = run.plan.launches * args.steps
    run.close()
    peak, peak_kind, _ = measured_peaks()
    achieved = BYTES_PER_PT["tti"] * npts / (kern_ms / 1e3) / 1e9
    value = npts * nt * args.steps / (ms / 1e3) / 1e9
    return {"metric": "GPts/s", "value": value, "unit": "GPts/s",
            "workload": "config3: 3D TTI p/r so=%d, %s (512^3 + 40 damping), "
                        "h=20 m, nt=%d%s"
                        % (so, "x".join(map(str, meta["shape"])), nt,
                           "" if nt == 500 else
                           " (short horizon of config 3's 500)"),
            "steps": args.steps, "ms_per_step": ms / args.steps,
            "ms_per_timestep": ms / args.steps / nt,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_pt": BYTES_PER_PT["tti"],
                         "kernel_ms_per_timestep": kern_ms,
                         "traffic": ncu_traffic("tti", so),
                         "traffic_unit": "bytes/time step, both passes (ncu "
                                         "dram read+write, profiles/"
                                         "traffic.json)",
                         "peak_kind": peak_kind},
            "gflops": value * FLOPS_PER_PT["tti"](so),
            "gpu_launches": int(launches),
            "kernels": rep_kernels(sec),
            "clocks": clk.summary()}


def rep_kernels(sec) -> dict:
    return {"dense_exec": sec.get("dense_exec"),
            "stage_ms": {k: v * 1e3 for k, v in sec["stages"].items()}}


def launches_per_step(rk) -> int:
    """Kernels one rank launches per time step (split steps launch the
    boundary planes, the early sources, the interior and the rest apart;
    the TTI dense stage is two passes)."""
    plan = rk.run.plan
    ndense = sum(1 for k in range(plan.nstages) if plan.stages[k] < 100)
    nsparse = plan.nstages - ndense
    per_dense = 2 if any(plan.dense[i].fast_kind == 3
                         for i in range(plan.ndense)) else 1
    if rk.overlap is None:
        return ndense * per_dense + nsparse
    ov = rk.overlap
    lo, hi = ov["interior"]
    n = (len(ov["early"]) + (1 if hi >= lo else 0)) * per_dense
    return n + nsparse + (1 if ov["n_early"] else 0)


def run_slabs(args, world, rank, local):
    """N GPUs: config 2 weak-scaled along x (config-4 layout), one x-slab
    per rank, ghost planes exchanged with NCCL send/recv every time step."""
    import torch
    import torch.distributed as dist
    import workloads
    from paper_1807_03032_b200.backend.slab import SlabRank, step_loop
    if args.workload == "config5":       # TTI so=12 strong scaling
        args.op, args.so = "tti", 12
        if args.nt == 500:
            args.nt = 300                # config 5's own nt
        op, bufs, dt, meta = workloads.config5_slab(world, rank, nt=args.nt)
    elif args.op == "tti":
        op, bufs, dt, meta = workloads.tti_weak_slab(
            world, rank, so=args.so, n=args.n, nt=args.nt)
    elif args.workload == "config4":
        if args.nt == 500:
            args.nt = 200                # config 4's own nt
        op, bufs, dt, meta = workloads.config4_slab(
            world, rank, so=args.so, n=1024 if args.n == 512 else args.n,
            nt=args.nt)
    else:
        op, bufs, dt, meta = workloads.weak_slab_problem(
            world, rank, so=args.so, n=args.n, nt=args.nt)
    from paper_1807_03032_b200.backend.slab import attach_native, make_comm
    ov = "force" if os.environ.get("SC_FORCE_SPLIT") else not args.no_overlap
    rk = SlabRank(op, bufs, rank, world, args.nt, device=local, dt=dt,
                  overlap=ov)
    # the library's data plane (sc_multi_run: boundary planes, NCCL ghost
    # exchange on a comm stream, interior, one CUDA graph per rank) unless
    # SC_MULTI_PY=1 selects the host-driven torch.distributed loop
    native = not os.environ.get("SC_MULTI_PY")
    comm = make_comm(rank, world) if native and world > 1 else None
    if native:
        attach_native(rk, comm)
    npts = int(np.prod(meta["shape"]))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def maxr(x):
        if world > 1:
            t = torch.tensor([x], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    for _ in range(args.warmup):
        step_loop(rk)
    # host cost of issuing a time step (must stay below its device time):
    # 32 steps, few enough that the launch queue never fills
    from paper_1807_03032_b200.backend.slab import step_once
    torch.cuda.synchronize()
    t_m, t_M = int(rk.env["t_m"]), int(rk.env["t_M"])
    host_ms = None
    if not native:
        probe = range(t_m, min(t_m + 32, t_M + 1))
        h0 = time.perf_counter()
        for t in probe:
            step_once(rk, t)
        host_ms = (time.perf_counter() - h0) * 1e3 * args.nt / \
            max(len(probe), 1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step_loop(rk)
        e1.record()
        barrier()
    ms = maxr(e0.elapsed_time(e1))
    value = npts * args.nt * args.steps / (ms / 1e3) / 1e9
    # per-stage times of this rank's slab (profiled pass)
    rep = rk.run.run(profile=True)
    stages = [v for v in rep.values() if "stages" in v][0]["stages"]
    dense_s = [v for k, v in stages.items() if k.startswith("dense")][0]
    slab_pts = (rk.b - rk.a) * meta["shape"][1] * meta["shape"][2]
    kern_ms = dense_s * 1e3 / args.nt
    achieved = BYTES_PER_PT[args.op] * slab_pts / (kern_ms / 1e3) / 1e9
    halo_overlap = rk.overlap is not None
    launches = launches_per_step(rk)
    # release this rank's device buffers before the end-to-end rank is built
    # (config 5 fills most of the GPU)
    rk.run.close()
    del rk
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    # end to end: build the rank (H2D of its window), run, gather (D2H)
    barrier()
    t0 = time.perf_counter()
    rk2 = SlabRank(op, bufs, rank, world, args.nt, device=local, dt=dt,
                   overlap=ov)
    if native:
        attach_native(rk2, comm)
    step_loop(rk2)
    rk2.run.download(xrange=rk2.owned_storage())
    barrier()
    e2e_s = maxr(time.perf_counter() - t0)
    peak, peak_kind, _ = measured_peaks()
    line = {
        "metric": "GPts/s", "value": value, "unit": "GPts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload == "config5" else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": ("synthetic (two-layer velocity, eps/delta/theta/phi "
                 "Gaussian-smoothed on the GPU from per-plane seeded noise, "
                 "one Ricker source, %d receivers)" % meta["nrec"]
                 if args.workload == "config5" else
                 "synthetic (config-3 cubes stacked in x: two-layer "
                 "velocity, Gaussian-smoothed eps/delta/theta/phi, one "
                 "Ricker source per slab)" if args.op == "tti" else
                 "synthetic (config-2 slabs stacked in x, one Ricker source "
                 "per slab, %d receivers)" % meta["nrec"]
                 if args.workload == "config2" else
                 "synthetic (two-layer velocity, zero damping field, one "
                 "Ricker source per slab, no receivers)"),
        "config": {"workload": ("config5 TTI strong scaling (1536x1024x1024 + "
                                "40 damping over all GPUs, 1024^2 receivers): "
                                if args.workload == "config5" else
                                "config3 TTI weak-scaled in x: "
                                if args.op == "tti" else
                                "config2 weak-scaled in x (config-4 layout): "
                                if args.workload == "config2" else
                                "config4 (1024^3 interior per GPU): ") +
                   "%s so=%d, global %s, nt=%d, x-slab per GPU, %d ghost "
                   "planes/side via NCCL send/recv" % (
                       args.op, args.so, "x".join(map(str, meta["shape"])),
                       args.nt, args.so // 2),
                   "label": workload_label(args, meta["shape"])
                   if args.workload == "config4" else None,
                   "operator": args.op,
                   "so": args.so, "grid": list(meta["shape"]), "nt": args.nt,
                   "parallelism": "x-slabs over %d GPUs" % world,
                   "halo_overlap": halo_overlap,
                   "data_plane": ("library: sc_multi_run (NCCL send/recv "
                                  "inside one CUDA graph per rank)"
                                  if native else
                                  "host-driven torch.distributed loop "
                                  "(SC_MULTI_PY=1)"),
                   "nccl": {"version": ".".join(map(str, torch.cuda.nccl.version())),
                            "comm": "sc_multi_init world=%d" % world
                            if comm is not None else None},
                   "host_issue_ms_per_timestep":
                       host_ms / args.nt if host_ms is not None else None},
        "gflops": value * FLOPS_PER_PT[args.op](args.so),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.op, args.so)
                     if world == 1 and args.workload == "config2" else None,
                     "traffic_unit": "bytes/launch (ncu dram read+write, "
                                     "profiles/traffic.json)",
                     "kernel": "%s so=%d on rank %d's slab (%.3f ms/launch)"
                               % ("acoustic_kernel" if args.op == "acoustic"
                                  else "tti passes", args.so, rank, kern_ms),
                     "peak_kind": peak_kind},
        "e2e": {"value": npts * args.nt / e2e_s / 1e9, "unit": "GPts/s",
                "h2d_bytes_per_step": rk2.run.h2d_bytes,
                "d2h_bytes_per_step": rk2.run.d2h_bytes},
        "gpu_launches": int(launches * args.nt * args.steps),
        "clocks": clk.summary(),
    }
    if args.workload == "config4":
        line["config"]["workload"] = line["config"].pop("label")
    else:
        line["config"].pop("label")
    if rank == 0:
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
