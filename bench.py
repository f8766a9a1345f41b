#!/usr/bin/env python
"""Benchmark of the B200 FoE/iPiano despeckling hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl foe|reference]

A *step* is one full pass of the hot path over one batch:
a1 init (w^0 = log max(f,1), F and grad F at w^0), `iters` iPiano iterations (inertial
step, Newton prox, energy + gradient at the candidate, backtracking decision), a13 output
u = e^w.  The metric is megapixel-iterations/s = images * H * W * iters / time (BASELINE.json
metric).  The Lipschitz initialisation (R-10) is setup, timed separately (lipschitz_ms).

Default workload: BASELINE.json configs[3] (c4) -- 64 independent 512x512 images per GPU
(L in {1,3,8}), 48 filters 7x7, 300 iterations -- weak scaling (N GPUs -> 64N images,
global image i keeps its seeds).  c4 is the configuration the FP32-roofline target and the
multi-GPU scaling target are quoted on.

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the
launching stream, with a 256 MiB L2 flush between steps (outside the events); barrier +
synchronize on both sides; max over ranks.  The fused prior-gradient kernel (K1) is timed
per launch with CUDA events on its own stream for the roofline entry.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixel-iterations/s of iPiano (FoE grad+prox) and % of B200 FP32 peak"
DTYPE_DETAIL = {1: "fp32 stencil (FFMA2), fp64 iterate/prox/reductions",
                2: "fp32-accurate stencil on tensor cores (tcgen05 kind::f16: fp16 x3 hi/lo split with "
                   "power-of-two scales, fp32 accumulate in TMEM), fp64 iterate/prox/reductions"}
UNIT = "MP-it/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["foe", "reference"], default="foe")
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--images", type=int, default=0, help="images per GPU (default: the config's batch)")
    ap.add_argument("--iters", type=int, default=0, help="override iteration count (quick runs only)")
    ap.add_argument("--stencil", choices=["auto", "ffma", "tensor"], default="auto",
                    help="prior kernel (auto: K8 tensor cores where it fills the GPU, else K1)")
    ap.add_argument("--solver", choices=["auto", "graph", "persistent"], default="auto",
                    help="trial-loop driver (auto: persistent for single small images, SURVEY 8(f) f4)")
    ap.add_argument("--filter-groups", type=int, default=0, help="K1 filter groups per tile (0: automatic)")
    ap.add_argument("--tile-rows", type=int, default=0, help="K8 output rows per tile (0: automatic)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-p2p", action="store_true", help="c5: ghost rows over ncclSend/Recv instead of K2 peer stores")
    ap.add_argument("--protocol", choices=["none", "fig2"], default="none",
                    help="fig2: the data-term protocol of the paper's Fig. 2 on synthetic data (GPU PSNR/SSIM of "
                         "models (8), (6), (10), lambda per model from a grid; paper_1404_5344_b200/fig2.py)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="c5: weak = a (1024 N) x 8192 scene, 1024 rows per GPU (SURVEY 8(d)); strong = the "
                         "fixed 8192^2 scene of BASELINE.json configs[4] cut into N slabs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=60,
                    help="oracle sample: iterations on one image (~10 s of host CPU work)")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram bytes per K1 launch from an ncu --set full capture (roofline.traffic)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            # wait (<= 3 s) for the sampler's first line, so that short timed regions (the small
            # configs: milliseconds) are covered too
            t0 = time.time()
            while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def smi_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].strip().isdigit():
            return int(ids[local_rank])
    return local_rank


# ------------------------------------------------------------------------- CPU oracle

def oracle_sample(cfg, d, iters):
    """Time the fp64 oracle (as it stands) on image 0 of the batch for `iters` iterations."""
    import oracle
    import foe_synth as S
    f = d["f"][0]
    l1, l2 = d["lambdas"][0]
    v0 = S.lipschitz_start_vector(1, cfg.H, cfg.W)[0]
    L0 = d.get("L0")
    L_init = float(L0[0]) if L0 is not None else 2.0 ** 18
    c = oracle.make_cfg(L_init, iters)
    t0 = time.perf_counter()
    run = oracle.ipiano_run(f, d["filters"], d["theta"], l1, l2, c)
    dt = time.perf_counter() - t0
    mp_it = cfg.H * cfg.W * iters / 1e6
    return dict(value=mp_it / dt, seconds=dt, cores=oracle.num_threads(), status=run["status"],
                sample=f"1 image {cfg.H}x{cfg.W} of {cfg.name}, {iters} iPiano iterations "
                       f"(+ initial gradient), fp64 C oracle, OpenMP over rows")


def run_reference(args, cfg):
    """--impl reference: the oracle as the reference arm (rank 0 only)."""
    import foe_synth as S
    from paper_1404_5344_b200 import dist as D
    rank, ws, local = D.world()
    if rank != 0:
        return 0
    d = S.make_inputs(cfg, images=[0])
    d["L0"] = None
    for _ in range(args.warmup):
        oracle_sample(cfg, d, 1)
    vals, secs = [], []
    for _ in range(args.steps):
        r = oracle_sample(cfg, d, args.cpu_iters)
        vals.append(r["value"]); secs.append(r["seconds"])
    value = len(vals) / sum(1.0 / v for v in vals)  # total MP-it / total time
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(cfg, 1, 1, cfg.H * cfg.W, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def roofline_entry(stencil, alg_tflops, k_ms, k_launches, step_ms, args, dev, cfg, persistent=False, tiling=None):
    """Roofline of the dominant kernel (the prior stencil, ~90% of the step).

    achieved = ALGORITHMIC flops (4 N_f m^2 per pixel per evaluation) / the
    kernel's event-timed duration.  K1 (FFMA2) is bound by the FP32 FMA pipes: peak = SMs x 128
    lanes x 2 x sm_max_mhz.  K8 (tcgen05 kind::f16, 3 passes for fp32 accuracy) runs on the tensor
    cores: peak = the measured sustained bf16 GEMM rate (fp16 and bf16 share the dense rate) -- the
    kernel is timed inside a long step; frac_fp32_emulated divides by peak / 3 (an fp32-accurate
    product costs three fp16 products); fp32_frac (against the FP32 FMA peak) is the BASELINE
    metric's "% of B200 FP32 peak"."""
    import torch
    peaks, peak_src = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = nsm * 128 * 2 * sm_max * 1e6 / 1e12
    micro = {}
    try:   # our own microbenchmarks (tools/probes/peaks.cu): FFMA2 chains, back-to-back tcgen05 TF32
        with open(os.path.join(ROOT, "profiles", "r01_peaks_microbench.json")) as fh:
            micro = json.load(fh)
    except Exception:
        pass
    traffic, traffic_src = args.traffic_bytes, "--traffic-bytes" if args.traffic_bytes else None
    if traffic is None:   # DRAM bytes per launch from the committed ncu --set full capture of this kernel
        try:
            with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
                tr = json.load(fh)
            key = "persistent" if persistent else ("k8" if stencil == 2 else "k1")
            if key in tr and (cfg.name == tr[key].get("config")):
                traffic, traffic_src = tr[key]["bytes_per_launch"], tr[key]["source"]
        except Exception:
            pass
    common = {"achieved": alg_tflops, "unit": "TFLOP/s", "traffic": traffic, "traffic_source": traffic_src,
              "fp32_peak": fp32_peak, "fp32_frac": (alg_tflops / fp32_peak) if alg_tflops else None,
              "k_ms_per_launch": k_ms / max(k_launches, 1), "k_launches": k_launches,
              "k_share_of_step": (k_ms / sum(step_ms)) if step_ms else None}
    if stencil == 2:
        bf16 = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)))
        m, nf = cfg.m, cfg.n_filters
        np_ = ((nf + 15) // 16) * 16
        nb = ((m * m // 8) * 8 + 15) // 16 * 16
        kf = ((m + 1) // 2) * 16                         # forward K: (m + 1) ring slots of 8 halves
        c = (m - 1) // 2
        R, ow, mode = tiling if tiling else (64, 128 - 2 * c, 0)
        rows = R if mode >= 1 else R + 2 * c          # response rows per tile (no row halos: R)
        # executed tensor flops per output pixel: 3 passes x 2 x (fwd Kf x NP + bwd NP x NB) per
        # response pixel, x `rows` 128-lane response rows per R x OW output tile (ipiano_state_tiling)
        exec_px = 3 * 2 * (kf * np_ + np_ * nb) * rows * 128 / (R * ow)
        alg_px = 4.0 * nf * m * m
        ex = alg_tflops * exec_px / alg_px if alg_tflops else None
        if micro.get("fp32_tflops", -1) > 0:
            common["fp32_peak_microbench"] = micro["fp32_tflops"]
        return dict(common, bound="tensor", peak=bf16, frac=(alg_tflops / bf16) if alg_tflops else None,
                    kernel="k_prior_grad_th (K8: tcgen05 kind::f16 x3, A operands and accumulators in TMEM)",
                    peak_source=f"measured: sustained bf16 GEMM {bf16:.1f} TFLOP/s ({peak_src} MEASURED_PEAKS.json; "
                                f"fp16 dense = bf16 dense rate)",
                    peak_fp32_emulated=bf16 / 3.0,
                    frac_fp32_emulated=(3.0 * alg_tflops / bf16) if alg_tflops else None,
                    tensor_executed_tflops=ex, tensor_executed_frac=(ex / bf16) if ex else None,
                    executed_per_algorithmic=exec_px / alg_px,
                    tiling={"tile_rows": R, "tile_cols": ow, "halo_mode": mode,
                            "halo_modes": "0 row+column halos, 1 no row halos, 2 neither (DESIGN.md 5, K8)"})
    kname = ("k_ipiano_persistent (all trial rounds of a solve in one cooperative launch: K2 + K1 FFMA2 "
             "stencil + K3 per round; timed around ipiano_solve, so achieved covers the whole round)"
             if persistent else "k_prior_grad2 (K1: FFMA2 fused FoE energy+gradient stencil)")
    return dict(common, bound="alu", peak=fp32_peak, frac=(alg_tflops / fp32_peak) if alg_tflops else None,
                kernel=kname,
                peak_source=f"derived: {nsm} SMs x 128 FP32 lanes x 2 flop x {sm_max:.0f} MHz "
                            f"(sm_max_mhz, {peak_src} MEASURED_PEAKS.json) -- DESIGN.md")


def config_block(cfg, n_gpus, images_per_gpu, px, args):
    iters = args.iters or cfg.iters
    return {
        "workload": f"{cfg.name}: {cfg.description}" + (f" [iters overridden to {iters}]" if args.iters else ""),
        "images_per_gpu": images_per_gpu, "global_images": images_per_gpu * n_gpus,
        "H": cfg.H, "W": cfg.W, "filters": f"{cfg.n_filters}x{cfg.m}x{cfg.m}", "iters": iters,
        "policy": "iPiano beta=0.4, a=0.95*2(1-b)/L_n, doubling backtracking, L nondecreasing, "
                  "L_init=2^ceil(log2 rho_hat) (DESIGN.md R-9/R-10)",
        "l2": "256 MiB buffer written between timed steps (outside the events)",
        "parallelism": f"dp{n_gpus} (independent images, no data-path collective)",
    }


# ------------------------------------------------------------------------------ main

_JSON_OUT = None


def emit(line: dict):
    """The one JSON line of this run, on the process's real stdout."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _isolate_stdout():
    """Send everything else written to fd 1 (NCCL's version banner, library prints) to stderr,
    so that stdout carries exactly the one JSON line the driver parses."""
    global _JSON_OUT
    try:
        sys.stdout.flush()
        real = os.dup(1)
        os.dup2(2, 1)
        _JSON_OUT = os.fdopen(real, "w")
    except OSError:
        _JSON_OUT = None


def main():
    _isolate_stdout()
    args = parse_args()
    import foe_synth as S
    cfg = S.config(args.config)
    if args.iters:
        cfg = S.config(args.config, iters=args.iters)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.protocol == "fig2":
        from paper_1404_5344_b200 import fig2
        res = fig2.run(iters=args.iters or 300)
        emit({"protocol": "fig2", "image": res["image"], "noisy": {"psnr": res["noisy"][0], "ssim": res["noisy"][1]},
              "models": {n: {"lambda": list(m["lam"]), "psnr": m["psnr"], "ssim": m["ssim"]}
                         for n, m in res["models"].items()},
              "note": "GPU runs, PSNR/SSIM by foe_psnr/foe_ssim; the fp64 oracle check of the chosen runs is "
                      "tests/test_fig2_protocol.py"})
        return 0
    if cfg.name == "c5":
        return run_slabs(args, cfg)

    import torch
    import paper_1404_5344_b200 as P
    from paper_1404_5344_b200 import dist as D

    rank, ws, local = D.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_img = args.images or cfg.B
    images = D.weak_shard(n_img, rank)
    d = S.make_inputs(cfg, images=images)
    B, H, W = d["f"].shape
    stream = torch.cuda.current_stream(dev)
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]), device=local)
    f_dev = torch.as_tensor(d["f"], device=dev)
    v0 = torch.as_tensor(S.lipschitz_start_vector(B, H, W), device=dev)

    # setup: Lipschitz initialisation (R-10), timed separately (a warm call: the first call of a
    # process also pays the lazy loading of the library's kernels, a one-time cost)
    rho, L0 = P.foe_estimate_lipschitz(md, f_dev, v0, 25)
    lipschitz_ms = lipschitz_timed(P, md, f_dev, v0, stream)
    d["L0"] = L0
    # (v0 stays: the e2e-with-setup leg re-runs the estimate)

    solver = {"auto": P.FOE_SOLVER_AUTO, "graph": P.FOE_SOLVER_GRAPH, "persistent": P.FOE_SOLVER_PERSISTENT}[args.solver]
    stencil = {"auto": P.FOE_STENCIL_AUTO, "ffma": P.FOE_STENCIL_FFMA, "tensor": P.FOE_STENCIL_TENSOR}[args.stencil]
    cfgc = P.ipiano_config_default(max_iters=cfg.iters, record_trace=0, solver=solver, stencil=stencil,
                                   filter_groups=args.filter_groups, tile_rows=args.tile_rows)
    st = P.ipiano_state_create(md, f_dev, d["lambdas"], L0, cfgc)
    u_dev = torch.empty((B, H, W), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    # small single-image configs resolve to the persistent driver (one cooperative launch per
    # solve); its dominant kernel is that launch, timed around ipiano_solve
    persistent = P.ipiano_state_solver(st) == P.FOE_SOLVER_PERSISTENT
    solve_ms = []

    def step(timed=False):
        P.ipiano_state_reset(st, f_dev, L0)
        if timed and persistent:
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            P.ipiano_solve(st)
            s1.record(stream)
            solve_ms.append((s0, s1))
        else:
            P.ipiano_solve(st)
        P.ipiano_get_iterate(st, want_w=False, u_out=u_dev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (value): inputs resident in HBM.  The dominant kernel's launches are
    # bracketed by CUDA events inside the timed region when they are long (>= 4 Mpx per launch:
    # c4, c5 -- the events cost nothing there); for short launches (c3: 37 us) events between
    # launches would break the CUDA graph and the programmatic launch overlap of the production
    # path, so the timed steps run the production path and one extra, profiled step after the
    # timed region gives the per-launch duration (config["kernel_timing"] says which)
    profile_in_timed = (not persistent) and B * H * W >= (1 << 22)
    if profile_in_timed:
        P.ipiano_profile(st, True)
        P.ipiano_profile_read(st)  # reset counters
        P.ipiano_profile_read_k2(st)
    sampler = ClockSampler(smi_index(local)) if rank == 0 else None
    if sampler:
        sampler.start()
    D.barrier()
    torch.cuda.synchronize()
    launches0 = P.foe_kernel_launches()
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(timed=True)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = P.foe_kernel_launches() - launches0
    D.barrier()
    clocks = sampler.stop() if sampler else None
    cnt = P.ipiano_get_counters(st)
    k2_ms, k2_launches = 0.0, 0
    if persistent:
        k1_ms, k1_launches = sum(a.elapsed_time(b) for a, b in solve_ms), len(solve_ms)
        kernel_timing = "the cooperative launch of each timed step, CUDA events on the launching stream"
    elif profile_in_timed:
        k1_ms, k1_launches, _ = P.ipiano_profile_read(st)
        k2_ms, k2_launches = P.ipiano_profile_read_k2(st)
        kernel_timing = "every launch in the timed region, CUDA events on the library's stream"
        # the same steps on the production launch path (CUDA graphs of programmatic launches, no
        # per-launch events), timed after the region: the per-launch events cost nothing here
        P.ipiano_profile(st, False)
        prod_ms = []
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            prod_ms.append(e0.elapsed_time(e1))
        prod_total = D.max_over_ranks(sum(prod_ms), dev)
        production_path = {"ms_per_step": prod_total / args.steps,
                           "value": D.sum_over_ranks(B * H * W * cfg.iters / 1e6 * args.steps, dev) / (prod_total / 1e3),
                           "path": "CUDA graph of programmatic dependent launches (no per-launch events), "
                                   "the same steps after the timed region"}
    else:
        P.ipiano_profile(st, True)
        P.ipiano_profile_read(st)
        P.ipiano_profile_read_k2(st)
        step()
        torch.cuda.synchronize()
        k1_ms, k1_launches, _ = P.ipiano_profile_read(st)
        k2_ms, k2_launches = P.ipiano_profile_read_k2(st)
        k1_ms *= args.steps           # per-launch time x the timed region's launches (same trials)
        k1_launches *= args.steps
        P.ipiano_profile(st, False)
        kernel_timing = ("one extra step after the timed region with CUDA events on the library's stream "
                         "(events between launches would break the graph/PDL path the timed steps use)")
    if not (profile_in_timed and not persistent):
        production_path = None
    total_ms = D.max_over_ranks(sum(step_ms), dev)
    mp_it_rank = B * H * W * cfg.iters / 1e6
    mp_it_total = D.sum_over_ranks(mp_it_rank * args.steps, dev)
    value = mp_it_total / (total_ms / 1e3)

    # K1 roofline: algorithmic flops = 4 N_f m^2 per pixel per evaluation;
    # evaluations in the timed region = trials (candidates) of every image, all steps
    trials_per_step = float(np.sum(cnt["trials"]))
    flops_per_eval_px = 4.0 * cfg.n_filters * cfg.m * cfg.m
    k1_flops = flops_per_eval_px * H * W * trials_per_step * args.steps
    k1_tflops = k1_flops / (k1_ms / 1e3) / 1e12 if k1_ms > 0 else None
    roofline = roofline_entry(P.ipiano_state_stencil(st), k1_tflops, k1_ms, k1_launches, step_ms, args, dev, cfg,
                              tiling=P.ipiano_state_tiling(st),
                              persistent=persistent)
    roofline["kernel_timing"] = kernel_timing
    fp32_peak = roofline["fp32_peak"]
    # K2 (inertial step + prox + partials), the second kernel of a round: HBM-bound at 32 B/px
    # algorithmic (read w, w- 8+8, g 4, f~ 4; write w+ 8), timed by the same events
    k2 = None
    if not persistent and k2_launches:
        k2_us = 1e3 * k2_ms / k2_launches
        k2_gbs = 32.0 * B * H * W / (k2_us * 1e-6) / 1e9
        hbm = measured_peaks()[0].get("hbm_gbs")
        k2 = {"us_per_launch": k2_us, "launches_profiled": k2_launches, "achieved_gbs": k2_gbs,
              "bytes_per_px": 32, "peak_gbs": hbm, "frac": (k2_gbs / hbm) if hbm else None}

    # ---- e2e: the public C-ABI call with host buffers (H2D of f and D2H of u inside)
    e2e = None
    if not args.no_e2e:
        f_pin = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)
        f_pin.copy_(torch.as_tensor(d["f"]))
        u_pin = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)
        f_np, u_np = f_pin.numpy(), u_pin.numpy()
        P.ipiano_run(md, f_np, d["lambdas"], L0, cfgc, u_out=u_np, want_trace=False)  # warm
        D.barrier()
        torch.cuda.synchronize()
        e2e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            P.ipiano_run(md, f_np, d["lambdas"], L0, cfgc, u_out=u_np, want_trace=False)
            e1.record(stream)
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
        D.barrier()
        e2e_total = D.max_over_ranks(sum(e2e_ms), dev)
        e2e = {"value": mp_it_total / (e2e_total / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(f_np.nbytes), "d2h_bytes_per_step": int(u_np.nbytes),
               "ms_per_step": e2e_total / args.steps,
               "call": "ipiano_run (C ABI) with pinned host f and u; state alloc + a1..a13 + copies"}
        # e2e with the required setup: H2D of f, the Lipschitz estimate (R-10: 25 power steps of
        # Hessian-vector products on the tensor cores), then ipiano_run with host buffers
        f_tmp = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        ews = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f_tmp.copy_(f_pin, non_blocking=True)
            _, L_s = P.foe_estimate_lipschitz(md, f_tmp, v0, 25)
            P.ipiano_run(md, f_np, d["lambdas"], L_s, cfgc, u_out=u_np, want_trace=False)
            e1.record(stream)
            e1.synchronize()
            ews.append(e0.elapsed_time(e1))
        D.barrier()
        ews_total = D.max_over_ranks(sum(ews), dev)
        e2e["with_setup"] = {"value": mp_it_total / (ews_total / 1e3), "unit": UNIT,
                             "ms_per_step": ews_total / args.steps,
                             "call": "H2D f + foe_estimate_lipschitz + ipiano_run (host f, u)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        r = oracle_sample(cfg, d, args.cpu_iters)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
               "sample": r["sample"], "seconds": r["seconds"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "dtype_detail": DTYPE_DETAIL[P.ipiano_state_stencil(st)],
            "data": "synthetic", "config": config_block(cfg, ws, B, H * W, args),
            "roofline": roofline, "k2": k2, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "trials_per_iter": trials_per_step / (B * cfg.iters),
            "run_fp32_frac": (flops_per_eval_px * H * W * trials_per_step * args.steps * ws / (total_ms / 1e3) / 1e12)
                             / fp32_peak / ws,
            "lipschitz_ms": lipschitz_ms, "status": [int(s) for s in set(cnt["status"].tolist())],
            "solver": "persistent" if persistent else "graph",
        }
        if production_path is not None:
            line["production_path"] = production_path
        emit(line)
    st.destroy()
    md.destroy()
    D.barrier()
    return 0


def lipschitz_timed(P, md, f_dev, v, stream, reps=3):
    """foe_estimate_lipschitz (R-10 setup) in ms: median of `reps` warm calls, CUDA events on the
    launching stream (the call synchronises it)"""
    import torch
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.foe_estimate_lipschitz(md, f_dev, v, 25)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def run_slabs(args, cfg):
    """c5 (BASELINE.json configs[4]): one SAR-like scene cut into N row slabs, one per GPU, with
    the per-trial 6-row ghost exchange and band-partial all-gather over NCCL (DESIGN.md
    "Multi-GPU").  --scaling weak (default): a (1024 N) x 8192 scene, 1024 rows per GPU (SURVEY
    8(d) "Scaling"); --scaling strong: the fixed 8192^2 scene.  A step = reset from f + `iters`
    iterations."""
    import torch
    import foe_synth as S
    import paper_1404_5344_b200 as P
    from paper_1404_5344_b200 import dist as D

    rank, ws, local = D.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.scaling == "weak":
        cfg = S.config("c5", H=1024 * ws, iters=cfg.iters)
    d = S.make_inputs(cfg)
    f_full = d["f"][0]
    Hg, W = f_full.shape
    r0, r1 = D.slab_rows(Hg, ws, rank)
    lam = tuple(d["lambdas"][0])
    md = P.foe_model_create(d["filters"], d["theta"], lam=lam, device=local)
    # setup: L_init (R-10) on the whole scene, identical on every rank (deterministic kernels)
    torch.cuda.synchronize()
    fw = torch.as_tensor(f_full[None], device=dev)
    v0 = torch.as_tensor(S.lipschitz_start_vector(1, Hg, W), device=dev)
    rho, L0 = P.foe_estimate_lipschitz(md, fw, v0, 25)          # warm call (lazy kernel loading)
    lipschitz_ms = lipschitz_timed(P, md, fw, v0, torch.cuda.current_stream(dev))
    del fw, v0
    L0 = float(L0[0])
    comm = P.foe_comm_create(D.share_bytes(P.foe_comm_unique_id() if rank == 0 else None), ws, rank, local)
    f_dev = torch.as_tensor(np.ascontiguousarray(f_full[r0:r1]), device=dev)
    stencil = {"auto": P.FOE_STENCIL_AUTO, "ffma": P.FOE_STENCIL_FFMA, "tensor": P.FOE_STENCIL_TENSOR}[args.stencil]
    cfgc = P.ipiano_config_default(max_iters=cfg.iters, record_trace=0, stencil=stencil)
    sl = P.ipiano_slabs_create(md, f_dev, Hg, lam=lam, lipschitz_init=L0, cfg=cfgc, comm=comm)
    # fused ghost-row exchange: K2 stores straight into the ring neighbours' ghost rows (CUDA IPC
    # over NVLink); the NCCL send/recv path stays if a mapping cannot be opened
    exchange = "ncclSend/Recv"
    if not args.no_p2p:
        import torch.distributed as dist
        h = P.ipiano_slabs_halo_handle(sl)
        hs = [h]
        if ws > 1:
            hs = [None] * ws
            dist.all_gather_object(hs, h)
        up, dn = D.ring_neighbours(rank, ws)
        ok = True
        try:
            P.ipiano_slabs_connect_peers(sl, hs[up], hs[dn])
        except P.FoeError as e:
            ok = False
            print(f"[bench] fused exchange unavailable on rank {rank}: {e}", file=sys.stderr)
        if D.all_true(ok):
            exchange = "K2 peer stores (CUDA IPC/NVLink) + NCCL ordering all-reduce"
        elif ok:
            P.ipiano_slabs_disconnect_peers(sl)      # every rank must take the same path
        P.ipiano_slabs_reset(sl, f_dev, L0)
    member = P.ipiano_slabs_member(sl, 0)
    u_dev = torch.empty((r1 - r0, W), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        P.ipiano_slabs_reset(sl, f_dev, L0)
        P.ipiano_slabs_solve(sl)
        P.ipiano_slabs_get_iterate(sl, want_w=False, u_out=u_dev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    P.ipiano_profile(member, True)
    P.ipiano_profile_read(member)
    sampler = ClockSampler(smi_index(local)) if rank == 0 else None
    if sampler:
        sampler.start()
    D.barrier()
    torch.cuda.synchronize()
    launches0 = P.foe_kernel_launches()
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = P.foe_kernel_launches() - launches0
    D.barrier()
    clocks = sampler.stop() if sampler else None
    k1_ms, k1_launches, _ = P.ipiano_profile_read(member)
    cnt = P.ipiano_get_counters(member)
    total_ms = D.max_over_ranks(sum(step_ms), dev)
    mp_it_total = Hg * W * cfg.iters * args.steps / 1e6
    value = mp_it_total / (total_ms / 1e3)
    trials_per_step = float(cnt["trials"][0])
    flops_px = 4.0 * cfg.n_filters * cfg.m * cfg.m
    k1_flops = flops_px * (r1 - r0) * W * trials_per_step * args.steps
    k1_tflops = k1_flops / (k1_ms / 1e3) / 1e12 if k1_ms > 0 else None
    roof = roofline_entry(P.ipiano_state_stencil(member), k1_tflops, k1_ms, k1_launches, step_ms, args, dev, cfg,
                          tiling=P.ipiano_state_tiling(member))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "dtype_detail": DTYPE_DETAIL[P.ipiano_state_stencil(member)], "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.description}" + (
                           f" (weak scaling: {Hg} x {W} scene, 1024 rows per GPU)" if args.scaling == "weak" else ""),
                       "H": Hg, "W": W,
                       "filters": f"{cfg.n_filters}x{cfg.m}x{cfg.m}", "iters": cfg.iters,
                       "slab_rows_per_gpu": r1 - r0,
                       "l2": "inputs (8192^2 fp64 state, 1.6 GB) larger than L2; 256 MiB flush between steps",
                       "parallelism": f"row slabs x{ws}: 6-row ghost exchange ({exchange}) + band all-gather per trial"},
            "roofline": roof,
            "cpu_baseline": None, "e2e": None, "gpu_launches": int(launches), "clocks": clocks,
            "trials_per_iter": trials_per_step / cfg.iters, "lipschitz_ms": lipschitz_ms,
            "status": [int(cnt["status"][0])],
        }
        emit(line)
    sl.destroy()
    comm.destroy()
    md.destroy()
    D.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
