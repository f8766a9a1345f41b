"""The Fig. 2 data-term protocol (paper_1404_5344_b200/fig2.py) on the GPU, with
each model's chosen run redone by the fp64 oracle: the three models (8), (6) and (10) on a seeded
image with L = 8 speckle, lambda per model by the best PSNR on a small grid (256^2 here so the
oracle's three 300-iteration runs take under a minute; `bench.py --protocol fig2` runs 512^2).  Per model: GPU
vs oracle final image relative L2 <= 1e-4 and |dPSNR| <= 0.01 dB (the P3 bars); PSNR/SSIM of the
library's kernels against the oracle's metrics to 1e-6 / 1e-5.  The table goes to $FIG2_OUT if set
(profiles/r02_fig2.json is such a run).  The paper's ordering (10) > (8) > (6) is NOT asserted:
it was measured with the learned filter bank, which is not available."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import metrics as OM  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402
from paper_1404_5344_b200 import fig2  # noqa: E402


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_fig2_protocol_against_oracle():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    H = W = int(os.environ.get("FIG2_SIZE", "256"))
    res = fig2.run(iters=300, H=H, W=W)
    clean, f, k, th = fig2.inputs(H, W)
    table = {"image": res["image"], "noisy": {"psnr": res["noisy"][0], "ssim": res["noisy"][1]}, "models": {}}
    assert res["noisy"][0] == pytest.approx(OM.psnr(f, clean), abs=1e-6)
    for name, m in res["models"].items():
        l1, l2 = m["lam"]
        c = oracle.make_cfg(m["L0"], 300)
        ref = oracle.ipiano_run_u(f, k, th, l1, c) if name == "(6)" else oracle.ipiano_run(f, k, th, l1, l2, c)
        assert ref["status"] == 0, name
        err = rel_l2(m["u"], ref["u"])
        ps_o, ss_o = OM.psnr(ref["u"], clean), OM.ssim(ref["u"], clean)
        table["models"][name] = {"lambda": [l1, l2], "L_init": m["L0"], "psnr_gpu": m["psnr"], "ssim_gpu": m["ssim"],
                                 "psnr_oracle": ps_o, "ssim_oracle": ss_o, "rel_l2_gpu_vs_oracle": err,
                                 "grid": [{"lambda": list(g[0]), "psnr": g[1], "ssim": g[2]} for g in m["grid"]]}
        assert err <= 1e-4, (name, err)
        assert abs(m["psnr"] - ps_o) <= 0.01, name
        assert m["psnr"] == pytest.approx(OM.psnr(m["u"], clean), abs=1e-5)
        assert m["ssim"] == pytest.approx(OM.ssim(m["u"], clean), abs=1e-5)
        assert m["psnr"] > res["noisy"][0]          # every model restores (directional check only)
    out = os.environ.get("FIG2_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(table, fh, indent=1)
