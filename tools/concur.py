"""Experiment: c4's 64 images as 1 state vs G states solved concurrently (G host threads, G
streams) -- does K2 of one half-batch overlap K8 of the other?  python tools/concur.py"""
import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import foe_synth as S
import paper_1404_5344_b200 as P

cfg = S.config("c4")
d = S.make_inputs(cfg)
B = cfg.B
dev = torch.device("cuda", 0)
md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]), device=0)
f_dev = torch.as_tensor(d["f"], device=dev)
v0 = torch.as_tensor(S.lipschitz_start_vector(B, cfg.H, cfg.W), device=dev)
_, L0 = P.foe_estimate_lipschitz(md, f_dev, v0, 25)
cfgc = P.ipiano_config_default(max_iters=cfg.iters, record_trace=0)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.iters
cfgc.max_iters = iters


def run(G, reps=3):
    n = B // G
    states = [P.ipiano_state_create(md, f_dev[g * n:(g + 1) * n], d["lambdas"][g * n:(g + 1) * n], L0[g * n:(g + 1) * n], cfgc)
              for g in range(G)]
    streams = [torch.cuda.Stream(dev) for _ in range(G)]

    def solve(g):
        with torch.cuda.stream(streams[g]):
            P.ipiano_state_reset(states[g], f_dev[g * n:(g + 1) * n], L0[g * n:(g + 1) * n], stream=streams[g])
            P.ipiano_solve(states[g], stream=streams[g])

    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=solve, args=(g,)) for g in range(G)]
        for t in th: t.start()
        for t in th: t.join()
        torch.cuda.synchronize()
        if r: ts.append(time.perf_counter() - t0)
    ms = 1e3 * min(ts)
    print(f"G={G}: {ms:.1f} ms per solve of {B} images, {B * cfg.H * cfg.W * iters / ms / 1e3:.0f} MP-it/s", flush=True)
    for s in states: P.ipiano_state_destroy(s)


for G in (1, 2, 4, 1, 2):
    run(G)
