#!/usr/bin/env python
"""Markdown summary of one evidence run (tools/gpu_final.sh TAG bench, plus ncu captures) for
profiles/ -- run here on the files gpurun brought back:

    python tools/evidence_summary.py gpurun_out/TAG [ncu reports ...] > profiles/rNN_summary.md
"""
import contextlib
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402


def line(path):
    try:
        return json.loads(open(path).read().strip().split("\n")[-1])
    except (OSError, ValueError, IndexError):
        return None


def fmt(x, nd=1):
    return "—" if x is None else (f"{x:.{nd}f}" if isinstance(x, float) else str(x))


def main():
    d = sys.argv[1]
    reps = sys.argv[2:]
    rows = [("c4 (default bench, BASELINE configs[3])", "bench.json"), ("c5 weak (1024 x 8192 per GPU, N=1)", "bench_c5_weak.json"),
            ("c5 strong (8192^2, 1 GPU)", "bench_c5_strong.json"), ("c1 (128^2, persistent FFMA driver)", "bench_c1.json"),
            ("c2 (256^2, graph + K8 4-row tiles)", "bench_c2.json"), ("c3 (512^2, graph + K8 8-row tiles)", "bench_c3.json"),
            ("reference arm (fp64 oracle, host cores)", "bench_ref.json")]
    print(f"# Evidence run `{os.path.basename(d.rstrip('/'))}` (one B200, `tools/gpu_final.sh`)\n")
    smoke = os.path.join(d, "smoke.log")
    if os.path.exists(smoke):
        print("Smoke: `" + open(smoke).read().strip().split("\n")[-1] + "`\n")
    print("`value` = images x H x W x iterations / device time (MP-it/s), inputs resident in HBM; `e2e` through "
          "`ipiano_run` with pinned host buffers; `with setup` adds H2D + `foe_estimate_lipschitz`; `graph path` = the "
          "same steps on the production launch path (CUDA graph of programmatic launches, no per-launch events).\n")
    print("| config | value | ms/step | graph path | e2e | e2e with setup | dominant kernel ms/launch | frac (peak) | "
          "K2 us/launch | lipschitz ms | SM MHz, reasons |")
    print("|---|---:|---:|---:|---:|---:|---|---:|---:|---:|---|")
    for name, f in rows:
        L = line(os.path.join(d, f))
        if not L:
            continue
        r = L.get("roofline") or {}
        e = L.get("e2e") or {}
        c = L.get("clocks") or {}
        pp = L.get("production_path") or {}
        kern = (r.get("kernel") or "").split(" ")[0]
        kms = r.get("k_ms_per_launch")
        frac = r.get("frac")
        fe = r.get("frac_fp32_emulated")
        fr = "—" if frac is None else f"{frac:.3f}" + (f" ({fe:.3f} fp32-emul.)" if fe else "")
        print(f"| {name} | **{fmt(L.get('value'))}** | {fmt(L.get('ms_per_step'), 2)} | {fmt(pp.get('value'))} | "
              f"{fmt(e.get('value'))} | {fmt((e.get('with_setup') or {}).get('value'))} | "
              f"{kern} {fmt(kms, 4)} | {fr} | {fmt((L.get('k2') or {}).get('us_per_launch'))} | "
              f"{fmt(L.get('lipschitz_ms'))} | {fmt(c.get('sm_mhz'), 0)} {c.get('reasons', '')} |")
    L = line(os.path.join(d, "bench.json"))
    if L:
        r = L["roofline"]
        print(f"\nc4 roofline of `{r.get('kernel')}`: achieved {r['achieved']:.1f} TFLOP/s algorithmic "
              f"(9408 flop/px x 16.78 Mpx per launch / {r['k_ms_per_launch']:.4f} ms), peak {r['peak']} "
              f"({r.get('peak_source')}): frac {r['frac']:.3f}; fp32-emulated peak (/3) frac "
              f"{r.get('frac_fp32_emulated', 0):.3f}; executed tensor flops {r.get('executed_per_algorithmic', 0):.2f}x "
              f"algorithmic; vs the FP32 FMA peak {r.get('fp32_frac', 0):.2f}x.  DRAM traffic per launch "
              f"{r.get('traffic')} B ({r.get('traffic_source')}).")
        if L.get("k2"):
            k = L["k2"]
            print(f"\nK2: {k['us_per_launch']:.1f} us per launch, {k['achieved_gbs']:.0f} GB/s algorithmic "
                  f"({k['bytes_per_px']} B/px) = {k['frac']:.3f} of {k['peak_gbs']} GB/s.")
    fig = line(os.path.join(d, "fig2.json"))
    if fig:
        print("\nFig. 2 protocol (`bench.py --protocol fig2`): `" + json.dumps(fig.get("models", fig))[:600] + "`")
    lc = os.path.join(d, "launches.csv")
    if os.path.exists(lc):
        print("\n## Launch list of the default bench command (`ncu --metrics gpu__time_duration.sum`, serialised, "
              "cold cache; includes the Lipschitz setup)\n")
        ncu_summary.launches(lc)
    if reps:
        print("\n## ncu --set full captures\n")
        for p in reps:
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                ncu_summary.report(p)
            print(buf.getvalue())


if __name__ == "__main__":
    main()
