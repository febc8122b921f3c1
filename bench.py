"""bench.py — HGMR registration throughput on B200 (contract: one JSON line).

Workload (N = 1): BASELINE.json configs[1] = C2, a Kinect-sized 320x240
synthetic depth-frame pair (76,800 points each), adaptive:3 (depth-3 GMM
tree, lambda_c = 0.01).  One STEP = one full frame-pair registration through
the reference's public API (register_clouds: tree build on the target + EM
on the source), as the paper times it.

* value  : registrations/s over all ranks, inputs already resident in HBM
           (device pointers), CUDA-event time per step on the library's stream,
           L2 flushed (256 MB write) before every timed step.
* e2e    : the same metric through the same C-ABI call with pinned HOST
           buffers: H2D of both clouds + all D2H result reads inside the timed
           region (host wall clock around each synchronous call).
* N > 1  : one process per GPU (torchrun), every rank registers its own copy of
           the C2 pair (independent pairs shard with no collective), weak
           scaling; value = N*K / max-over-ranks time.  The `c4` item is the
           1M-point scene point-sharded over the N ranks (NCCL all-reduces of
           the per-node records each exchange step; strong scaling).
* configs: the C1 and C3 pairs beside the headline (N = 1).
* --impl reference: the reference's own CPU implementation (oracle/_ref =
           /root/reference sources built with the test shims) on the host's
           cores, same workload and metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "registrations/sec + tree-build Mpoints/sec at 1/2/4/8 B200; HBM roofline frac"
UNIT = "registrations/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(cfg_name: str):
    from paper_1807_02587_b200 import treereg as tr
    if cfg_name == "c2":
        tg, sr, gt = tr.kinect_pair(2)
        return tg, sr, gt, 3, "C2 Kinect 320x240 synthetic depth-frame pair (76,800 pts each), adaptive:3"
    if cfg_name == "c3":
        tg, sr, gt = tr.lidar_pair(3)
        return tg, sr, gt, 3, "C3 HDL-32-style synthetic sweep pair (72,000 pts each), adaptive:3"
    if cfg_name == "c1":
        tg = tr.unit_normalized(tr.synthetic("lumpy", 10000, 1))
        T = tr.random_rigid_transform(15.0, 0.05, 1)
        sr = T(tg)
        return tg, sr, T.inverse(), 2, "C1 unit-normalized lumpy 10k pair, adaptive:2"
    raise SystemExit(f"unknown config {cfg_name}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def config_dict(wl: str, world: int):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": wl, "pairs_per_rank_per_step": 1,
            "l2": "GPU arm: flushed (256 MB write) before every timed step; CPU arm: n/a",
            "parallelism": f"independent pairs, one per rank per step, x{world} ranks, no collectives"}


def algorithmic_bytes(diag, n_target: int, n_source: int, J: int, em_iters: int):
    """FP64 (s = 8), entry = idx 4 B + w 8 B + point 24 B.
    Build: per round 36 passes over E_l entries + the partition write of
    E_{l+1}, plus P_cal calibration associations.  Registration: I_em E-steps."""
    s = 8
    ent = 12 + 3 * s
    E = list(diag.entries_per_round) + [0]
    L = len(diag.entries_per_round)
    b_rounds = sum(36 * E[l] * ent + E[l + 1] * ent for l in range(L))
    b_assoc_cal = n_target * 3 * s + J * 136 + J * 104
    b_build = b_rounds + diag.calibration_passes * b_assoc_cal
    b_assoc_reg = n_source * 3 * s + J * 136 + J * 32
    return b_build, em_iters * b_assoc_reg


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("TRG_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend)
    return world, rank, local, dist


def max_over_ranks(x: float, dist, device=None):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist, device=None):
    if dist is not None:
        import torch
        t = torch.zeros(1, device=device)
        dist.all_reduce(t)


# --------------------------------------------------------------- reference
def run_reference(args):
    world, rank, local, dist = dist_setup(args.gpus)
    if rank != 0:
        return 0
    from oracle.oracle import Ref  # the reference's own CPU implementation
    tg, sr, gt, L, wl = workload(args.config)
    ref = Ref()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    for _ in range(args.warmup):
        ref.register_clouds(tg, sr, level=L)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.register_clouds(tg, sr, level=L)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(wl, args.gpus),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} full registrations (build+EM) of the {args.config.upper()} pair"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    world, rank, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1807_02587_b200 import treereg as tr
    ctx = tr.Context(local)
    tg, sr, gt, L, wl = workload(args.config)
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", L))
    tg_d = torch.from_numpy(tg).to(dev).contiguous()
    sr_d = torch.from_numpy(sr).to(dev).contiguous()
    tg_h = torch.from_numpy(tg).pin_memory()
    sr_h = torch.from_numpy(sr).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def step_dev():
        return tr.register_clouds(tg_d, sr_d, cfg, ctx)

    def step_host():
        return tr.register_clouds(tg_h.numpy(), sr_h.numpy(), cfg, ctx)

    for _ in range(args.warmup):
        res = step_dev()
        step_host()
    torch.cuda.synchronize()
    # accuracy of the measured registration (vs the generator's ground truth)
    rot_err = float(np.degrees(np.arccos(np.clip(
        (np.trace(res.transform.rotation.T @ gt.rotation) - 1) / 2, -1, 1))))
    # ---- device-resident timing
    launches0 = ctx.kernel_launches
    step_ms, build_s, em_s = [], [], []
    barrier(dist, dev)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = step_dev()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            build_s.append(r.model_build_seconds)
            em_s.append(r.em_seconds)
        torch.cuda.synchronize()
    barrier(dist, dev)
    launches = (ctx.kernel_launches - launches0) / args.steps
    t_dev = max_over_ranks(sum(step_ms) / 1e3, dist, dev)
    # ---- end-to-end through the C-ABI with host buffers
    h0, d0 = ctx.transfer_bytes()
    e2e_s = []
    barrier(dist, dev)
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_host()
        e2e_s.append(time.perf_counter() - t0)
    h1, d1 = ctx.transfer_bytes()
    t_e2e = max_over_ranks(sum(e2e_s), dist, dev)
    n_total = world * args.steps
    value = n_total / t_dev
    e2e = n_total / t_e2e
    # ---- roofline of the dominant kernel (the build, k_build)
    diag = tr.BuildDiagnostics()
    tree = tr.build_tree(tg_d, tr.ModelConfig(max_level=L), diag, ctx)
    J = tree.size()
    b_build, b_em = algorithmic_bytes(diag, len(tg), len(sr), J, res.iterations)
    t_build = float(np.median(build_s))
    t_em = float(np.median(em_s))
    peak, peak_kind = load_peaks()
    achieved = b_build / t_build / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k_build_dram_bytes.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")  # ncu, same command
        except Exception:
            traffic = None
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl, world),
        "tree_build_mpoints_per_s": world * len(tg) / t_build / 1e6,
        "phase_ms": {"build": 1e3 * t_build, "em": 1e3 * t_em,
                     "em_iterations": res.iterations, "converged": res.converged},
        "rot_err_deg_vs_gt": rot_err,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "tree build: k_build + k_calibrate (one launch each per step)",
                     "algorithmic_bytes": b_build, "peak_kind": peak_kind,
                     "E_per_round": list(diag.entries_per_round),
                     "calibration_passes": diag.calibration_passes},
        "e2e": {"value": e2e, "unit": UNIT,
                "h2d_bytes_per_step": (h1 - h0) // args.steps,
                "d2h_bytes_per_step": (d1 - d0) // args.steps},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if args.batch > 0:
        try:
            out["batched"] = run_batched(args, tr, ctx, cfg, dist, dev, world)
        except Exception as e:  # the headline line must survive a failing side item
            out["batched"] = {"error": f"{type(e).__name__}: {e}"}
    if args.c4:
        try:
            out["c4"] = run_c4(args, tr, ctx, dist, dev, world)
        except Exception as e:  # the headline line must survive a failing side item
            out["c4"] = {"error": f"{type(e).__name__}: {e}"}
    if args.extra and world == 1:
        try:
            out["configs"] = {c: run_small(tr, ctx, dev, c, args.steps) for c in ("c1", "c3") if c != args.config}
        except Exception as e:
            out["configs"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_c4(args, tr, ctx, dist, dev, world):
    """BASELINE C4: synthetic_scene(1M, seed 4), depth-4 tree, pose
    random_rigid_transform({8 deg, 0.03, seed 4}).  One GPU: the single-launch
    path.  N GPUs: every rank holds a contiguous 1/N block of both clouds and
    runs the point-sharded path (per-node records, leaf and EM moments
    all-reduced over NCCL each exchange step); the value is registrations of
    the whole cloud per second (strong scaling).  `parity`: the transform
    against the reference's own register_clouds on this pose
    (tests/golden/c4_scene1M_L4.npz), 1e-4 rad / 1e-4 x extent."""
    import torch
    pts = tr.synthetic("scene", 1_000_000, 4)
    T = tr.random_rigid_transform(8.0, 0.03, 4)
    src = (pts - T.translation) @ T.rotation
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 4))
    rank = dist.get_rank() if dist is not None else 0
    if world > 1:
        comm = tr.Comm.from_torch_distributed(ctx)
        lo, hi = tr.shard_bounds(len(pts), world, rank)
        tg = [torch.from_numpy(pts[lo:hi]).to(dev).contiguous()]
        sr = [torch.from_numpy(np.ascontiguousarray(src[lo:hi])).to(dev).contiguous()]
        step = lambda: tr.register_clouds_sharded(tg, sr, comm, cfg)  # noqa: E731
    else:
        tg = torch.from_numpy(pts).to(dev).contiguous()
        sr = torch.from_numpy(src).to(dev).contiguous()
        step = lambda: tr.register_clouds(tg, sr, cfg, ctx)  # noqa: E731
    res = step()
    torch.cuda.synchronize()
    reps = 2
    barrier(dist, dev)
    t0 = time.perf_counter()
    builds = []
    for _ in range(reps):
        res = step()
        builds.append(res.model_build_seconds)
    torch.cuda.synchronize()
    dt_all = max_over_ranks(time.perf_counter() - t0, dist, dev)
    ang = float(np.degrees(np.arccos(np.clip((np.trace(res.transform.rotation.T @ T.rotation) - 1) / 2,
                                             -1, 1))))
    parity = None
    try:
        z = np.load(os.path.join(ROOT, "tests", "golden", "c4_scene1M_L4.npz"))
        ext = float(np.linalg.norm(pts.max(0) - pts.min(0)))
        dr = float(np.arccos(np.clip((np.trace(res.transform.rotation.T @ z["rc_R"]) - 1) / 2, -1, 1)))
        dt = float(np.linalg.norm(res.transform.translation - z["rc_t"]))
        parity = {"vs": "reference register_clouds (golden)", "rot_rad": dr, "trans": dt,
                  "ok": bool(dr <= 1e-4 and dt <= 1e-4 * ext and res.iterations == int(z["rc_meta"][0]))}
    except Exception as e:  # fixture missing: report, don't fail
        parity = {"vs": "unavailable", "error": str(e)}
    roof = None
    if world == 1:  # the HBM fraction is meaningful at C4 (entries exceed L2)
        diag = tr.BuildDiagnostics()
        tree = tr.build_tree(tg, tr.ModelConfig(max_level=4), diag, ctx)
        b_build, _ = algorithmic_bytes(diag, len(pts), len(src), tree.size(), res.iterations)
        t_build = float(np.median(builds))
        peak, peak_kind = load_peaks()
        ach = b_build / t_build / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "kernel": "tree build (k_build + k_calibrate), C4", "algorithmic_bytes": b_build,
                "peak_kind": peak_kind, "E_per_round": list(diag.entries_per_round),
                "calibration_passes": diag.calibration_passes}
    return {"workload": "C4 synthetic_scene(1M, seed 4), adaptive:4" +
                        (f", point-sharded over {world} GPUs (NCCL)" if world > 1 else ", one GPU"),
            "scaling": "strong" if world > 1 else None,
            "value": reps / dt_all, "unit": UNIT, "ms_per_registration": 1e3 * dt_all / reps,
            "timing": "host wall clock around synchronous registrations, max over ranks",
            "tree_build_mpoints_per_s": len(pts) / float(np.median(builds)) / 1e6,
            "em_iterations": res.iterations, "converged": res.converged,
            "em_ms": 1e3 * res.em_seconds,
            "ms_per_em_iteration": 1e3 * res.em_seconds / max(1, res.iterations),
            "rot_err_deg_vs_gt": ang, "parity": parity, "roofline": roof, "ranks": world,
            "note": "the reference's own register_clouds does not converge on this pose either "
                    "(50 iterations, same answer: tests/test_c4_gpu.py)"}


def run_batched(args, tr, ctx, cfg, dist, dev, world):
    """C5 slice: `--batch` independent Kinect-sized pairs per rank (pair k
    uses noise and pose seed k), device-resident, through trg_register_batch:
    waves of `--streams` pairs in flight (0 = library default, 24), each wave's
    builds and EMs as single launches with one CTA group per pair.  Timed by
    the host clock around whole synchronous batches, max over ranks."""
    import torch
    rank = dist.get_rank() if dist is not None else 0
    # the pairs are rendered on the device (bit-identical to tr.kinect_pair)
    pairs = [tr.kinect_pair_device(1 + rank * args.batch + k, ctx) for k in range(args.batch)]
    tg = [p[0] for p in pairs]
    sr = [p[1] for p in pairs]
    for _ in range(1):
        tr.register_batch(tg, sr, cfg, ctx, args.streams)
    torch.cuda.synchronize()
    reps = max(1, min(3, args.steps))
    barrier(dist, dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        res = tr.register_batch(tg, sr, cfg, ctx, args.streams)
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, dist, dev)
    errs = [float(np.degrees(np.arccos(np.clip((np.trace(r.transform.rotation.T @ p[2].rotation) - 1) / 2,
                                               -1, 1)))) for r, p in zip(res, pairs)]
    out = {"workload": f"C5 slice: {args.batch} independent C2-style Kinect pairs per rank (seeds k)",
           "pairs_per_rank": args.batch, "pairs_in_flight": min(args.streams or 24, args.batch), "reps": reps,
           "value": world * args.batch * reps / dt, "unit": UNIT,
           "ms_per_batch": 1e3 * dt / reps, "timing": "host wall clock around synchronous batches",
           "converged": sum(r.converged for r in res), "median_rot_err_deg_vs_gt": float(np.median(errs))}
    # the same batch with the opt-in FP32 scoring of the EM (not
    # the parity mode above): rate, and the largest deviation from the FP64 answers
    fcfg = dataclasses.replace(cfg, fast_scoring=True)
    tr.register_batch(tg, sr, fcfg, ctx, args.streams)
    torch.cuda.synchronize()
    barrier(dist, dev)
    t0 = time.perf_counter()
    fres = tr.register_batch(tg, sr, fcfg, ctx, args.streams)
    torch.cuda.synchronize()
    fdt = max_over_ranks(time.perf_counter() - t0, dist, dev)
    devs = [float(np.arccos(np.clip((np.trace(a.transform.rotation.T @ b.transform.rotation) - 1) / 2, -1, 1)))
            for a, b in zip(res, fres) if a.converged and b.converged]
    out["fast_scoring"] = {"value": world * args.batch / fdt, "unit": UNIT,
                           "converged": sum(r.converged for r in fres),
                           "max_rot_dev_rad_vs_fp64_converged": max(devs) if devs else None,
                           "note": "opt-in FP32 scoring of the EM descent; deviations over the pairs both "
                                   "modes converge on (a non-converging EM wanders differently)"}
    return out


def cpu_baseline(cfg_name, samples: int = 5):
    """The reference implementation (oracle/_ref) on this host's cores: one
    warm-up registration of the same pair, then the median of `samples`
    timed ones (a bounded ~10 s sample), plus one serial (1-thread) run."""
    try:
        from oracle.oracle import Ref
        tg, sr, gt, L, wl = workload(cfg_name)
        ref = Ref()
        cores = os.cpu_count() or 1
        ref.set_threads(cores)
        ref.register_clouds(tg, sr, level=L)  # warm-up
        ts = []
        for _ in range(samples):
            t0 = time.perf_counter()
            ref.register_clouds(tg, sr, level=L)
            ts.append(time.perf_counter() - t0)
        dt = float(np.median(ts))
        # the reference's serial run beside the all-cores one
        ref.set_threads(1)
        t0 = time.perf_counter()
        ref.register_clouds(tg, sr, level=L)
        dt1 = time.perf_counter() - t0
        ref.set_threads(cores)
        return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"median of {samples} full registrations (build+EM) of the {cfg_name.upper()} "
                          f"pair after 1 warm-up, {cores} threads: {dt:.3f} s "
                          f"(min {min(ts):.3f}, max {max(ts):.3f})",
                "serial": {"value": 1.0 / dt1, "unit": UNIT, "cores": 1,
                           "sample": f"the same registration on 1 thread, {dt1:.2f} s"}}
    except Exception as e:  # the oracle build is test infrastructure; report, don't fail
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def run_small(tr, ctx, dev, cfg_name, steps):
    """BASELINE configs[0] (C1) / [2] (C3) beside the headline: device-resident
    registrations, CUDA events on the library's stream, L2 flushed per step."""
    import torch
    tg, sr, gt, L, wl = workload(cfg_name)
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", L))
    tg_d = torch.from_numpy(tg).to(dev).contiguous()
    sr_d = torch.from_numpy(sr).to(dev).contiguous()
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(3):
        res = tr.register_clouds(tg_d, sr_d, cfg, ctx)
    ms, bs = [], []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = tr.register_clouds(tg_d, sr_d, cfg, ctx)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        bs.append(res.model_build_seconds)
    ang = float(np.degrees(np.arccos(np.clip((np.trace(res.transform.rotation.T @ gt.rotation) - 1) / 2, -1, 1))))
    return {"workload": wl, "value": 1e3 * steps / sum(ms), "unit": UNIT,
            "ms_per_step": sum(ms) / steps, "build_ms": 1e3 * float(np.median(bs)),
            "em_iterations": res.iterations, "converged": res.converged, "rot_err_deg_vs_gt": ang}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=256, help="C5 slice: pairs per rank (0 = skip)")
    ap.add_argument("--streams", type=int, default=0,
                    help="C5 slice: pairs in flight per GPU (0 = library default)")
    ap.add_argument("--c4", type=int, default=1, help="add the C4 (1M points, depth 4) line item "
                    "(point-sharded over NCCL when N > 1)")
    ap.add_argument("--extra", type=int, default=1, help="add the C1 and C3 line items (N = 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
