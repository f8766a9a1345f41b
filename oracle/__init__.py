"""fp64 CPU oracle for the FoE/iPiano despeckling hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1404_5344_b200``) never imports it, and the
two share no code; the only common module is ``foe_synth`` (seeded inputs, no
method arithmetic).

Two tiers:
  * ``oracle.brute``  -- numpy, dense N x N operator matrices, for grids <= 16x16;
  * this module      -- ctypes wrapper over ``foe_oracle.c`` (plain C, fp64, OpenMP
                        over rows with fixed-order reductions) for the full configs.

Every function cites the PAPER.md passage it follows; see foe_oracle.c.
Functions with no independent pin are marked "parity unpinned" (none at present;
see DESIGN.md "Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "foe_oracle.c")
_BUILD = os.path.join(_HERE, "build")
_lock = threading.Lock()
_lib = None

ORC_OK, ORC_ERR_ARG, ORC_ERR_NONFINITE, ORC_ERR_BACKTRACK, ORC_ERR_PROX, ORC_ERR_DOMAIN = 0, 1, 4, 5, 6, 7
TR_FIELDS = 8
TRACE_NAMES = ("F", "G", "H", "L", "trials", "margin", "newton", "relchg")


def _so_path() -> str:
    with open(_SRC, "rb") as fh:
        h = hashlib.sha1(fh.read()).hexdigest()[:12]
    return os.path.join(_BUILD, f"liboracle_{h}.so")


def build(force: bool = False) -> str:
    """Compile foe_oracle.c with gcc (plain -O2, no fast-math, no FMA contraction)."""
    so = _so_path()
    if os.path.exists(so) and not force:
        return so
    os.makedirs(_BUILD, exist_ok=True)
    tmp = so + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-o", tmp, _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, so)
    return so


class OrcCfg(C.Structure):
    _fields_ = [
        ("beta", C.c_double), ("step_safety", C.c_double), ("lipschitz_init", C.c_double),
        ("backtrack_factor", C.c_double), ("shrink", C.c_double), ("max_iters", C.c_int),
        ("max_backtracks", C.c_int), ("newton_max_iters", C.c_int), ("newton_tol", C.c_double),
        ("rel_change_tol", C.c_double), ("w_guard", C.c_double),
    ]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            dp = C.POINTER(C.c_double)
            fp = C.POINTER(C.c_float)
            ip = C.POINTER(C.c_int)
            L.orc_conv.argtypes = [dp, C.c_int, C.c_int, dp, C.c_int, dp]
            L.orc_conv_adj.argtypes = [dp, C.c_int, C.c_int, dp, C.c_int, dp]
            for n in ("orc_rho", "orc_rho_prime", "orc_rho_second"):
                getattr(L, n).argtypes = [C.c_double]
                getattr(L, n).restype = C.c_double
            L.orc_energy_grad_u.argtypes = [dp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int, dp, dp]
            L.orc_energy_grad_w.argtypes = [dp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int, dp, dp]
            L.orc_hvp_w.argtypes = [dp, dp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int, dp]
            L.orc_data_energy.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, C.c_double]
            L.orc_data_energy.restype = C.c_double
            L.orc_prox_pixel.argtypes = [C.c_double] * 6 + [C.c_int, dp, dp]
            L.orc_prox.argtypes = [dp, dp, C.c_size_t, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_int, dp, dp, C.POINTER(C.c_longlong)]
            L.orc_ipiano_trial.argtypes = [dp, dp, dp, C.c_double, C.c_double, dp, C.c_int, C.c_int,
                                           dp, dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.POINTER(OrcCfg), dp, dp, dp, dp]
            L.orc_ipiano_run.argtypes = [fp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int,
                                         C.c_double, C.c_double, C.POINTER(OrcCfg), dp, dp, ip, ip]
            L.orc_estimate_lipschitz.argtypes = [fp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int,
                                                 dp, C.c_int, dp]
            L.orc_estimate_lipschitz.restype = C.c_double
            L.orc_idiv_energy.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double]
            L.orc_idiv_energy.restype = C.c_double
            L.orc_idiv_prox_pixel.argtypes = [C.c_double] * 4
            L.orc_idiv_prox_pixel.restype = C.c_double
            L.orc_hvp_u.argtypes = [dp, dp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int, dp]
            L.orc_ipiano_trial_u.argtypes = [dp, dp, dp, C.c_double, C.c_double, dp, C.c_int, C.c_int,
                                             dp, dp, C.c_int, C.c_int, C.c_double,
                                             C.POINTER(OrcCfg), dp, dp, dp, dp]
            L.orc_ipiano_run_u.argtypes = [fp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int, C.c_double,
                                           C.POINTER(OrcCfg), dp, dp, ip, ip]
            L.orc_estimate_lipschitz_u.argtypes = [fp, C.c_int, C.c_int, dp, dp, C.c_int, C.c_int,
                                                   dp, C.c_int, dp]
            L.orc_estimate_lipschitz_u.restype = C.c_double
            L.orc_num_threads.restype = C.c_int
            _lib = L
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ---------------------------------------------------------------------------- operators

def conv(u, k) -> np.ndarray:
    """(k * u), true periodic convolution (reading R-2/R-3)."""
    u, k = _d(u), _d(k)
    out = np.empty_like(u)
    lib().orc_conv(_ptr(u), u.shape[0], u.shape[1], _ptr(k), k.shape[0], _ptr(out))
    return out


def conv_adj(v, k) -> np.ndarray:
    """K^T v, the exact adjoint of ``conv``."""
    v, k = _d(v), _d(k)
    out = np.empty_like(v)
    lib().orc_conv_adj(_ptr(v), v.shape[0], v.shape[1], _ptr(k), k.shape[0], _ptr(out))
    return out


def rho(x: float) -> float:
    return lib().orc_rho(float(x))


def rho_prime(x: float) -> float:
    return lib().orc_rho_prime(float(x))


def rho_second(x: float) -> float:
    return lib().orc_rho_second(float(x))


def energy_grad_u(u, filters, theta, want_grad=True):
    """E_FoE(u) and grad_u (Eq.(2), :194-198)."""
    u, k, th = _d(u), _d(filters), _d(theta)
    F = C.c_double()
    g = np.empty_like(u) if want_grad else None
    lib().orc_energy_grad_u(_ptr(u), u.shape[0], u.shape[1], _ptr(k), _ptr(th), k.shape[0],
                            k.shape[1], C.byref(F), _ptr(g) if want_grad else None)
    return (F.value, g) if want_grad else F.value


def energy_grad_w(w, filters, theta, want_grad=True):
    """F(w) = E_FoE(e^w) and grad_w F = W sum theta_i K_i^T rho'(K_i e^w)."""
    w, k, th = _d(w), _d(filters), _d(theta)
    F = C.c_double()
    g = np.empty_like(w) if want_grad else None
    lib().orc_energy_grad_w(_ptr(w), w.shape[0], w.shape[1], _ptr(k), _ptr(th), k.shape[0],
                            k.shape[1], C.byref(F), _ptr(g) if want_grad else None)
    return (F.value, g) if want_grad else F.value


def hvp_w(w, v, filters, theta) -> np.ndarray:
    """Hessian-vector product of F(w) (reading R-10)."""
    w, v, k, th = _d(w), _d(v), _d(filters), _d(theta)
    out = np.empty_like(w)
    lib().orc_hvp_w(_ptr(w), _ptr(v), w.shape[0], w.shape[1], _ptr(k), _ptr(th), k.shape[0],
                    k.shape[1], _ptr(out))
    return out


def ftilde(f) -> np.ndarray:
    """f~ = max(f, 1) in fp64 (reading R-4)."""
    return np.maximum(np.asarray(f, np.float32).astype(np.float64), 1.0)


def data_energy(w, ft, l1, l2) -> float:
    """G(w) of Eq.(10)."""
    w, ft = _d(w), _d(ft)
    return lib().orc_data_energy(_ptr(w), _ptr(ft), w.shape[0], w.shape[1], float(l1), float(l2))


def prox_pixel(what, ft, tau, l1, l2, tol=1e-12, cap=30):
    """Scalar prox of Eq.(9)/(10) by safeguarded Newton."""
    z, r = C.c_double(), C.c_double()
    it = lib().orc_prox_pixel(float(what), float(ft), float(tau), float(l1), float(l2),
                              float(tol), int(cap), C.byref(z), C.byref(r))
    return z.value, it, r.value


def prox(what, ft, tau, l1, l2, tol=1e-12, cap=30):
    what, ft = _d(what), _d(ft)
    out = np.empty_like(what)
    mres = C.c_double()
    bad = C.c_longlong()
    it = lib().orc_prox(_ptr(what), _ptr(ft), what.size, float(tau), float(l1), float(l2),
                        float(tol), int(cap), _ptr(out), C.byref(mres), C.byref(bad))
    return out, it, mres.value


def make_cfg(lipschitz_init, max_iters, beta=0.4, step_safety=0.95, backtrack_factor=2.0,
             shrink=1.0, max_backtracks=60, newton_max_iters=30, newton_tol=1e-12,
             rel_change_tol=0.0, w_guard=40.0) -> OrcCfg:
    return OrcCfg(beta, step_safety, lipschitz_init, backtrack_factor, shrink, max_iters,
                  max_backtracks, newton_max_iters, newton_tol, rel_change_tol, w_guard)


def ipiano_trial(w, wprev, g, F, L, f, filters, theta, l1, l2, cfg: OrcCfg, want_gplus=True):
    """One iPiano trial.  Returns dict.  want_gplus=False
    skips grad F(w+) (the C routine's gplus output is optional: F(w+) alone decides the test)."""
    w, wprev, g = _d(w), _d(wprev), _d(g)
    ft = ftilde(f)
    k, th = _d(filters), _d(theta)
    what = np.empty_like(w)
    wplus = np.empty_like(w)
    gplus = np.empty_like(w) if want_gplus else None
    out = np.empty(8)
    st = lib().orc_ipiano_trial(_ptr(w), _ptr(wprev), _ptr(g), float(F), float(L), _ptr(ft),
                                w.shape[0], w.shape[1], _ptr(k), _ptr(th), k.shape[0], k.shape[1],
                                float(l1), float(l2), C.byref(cfg), _ptr(what), _ptr(wplus),
                                _ptr(gplus) if want_gplus else None, _ptr(out))
    return dict(status=st, what=what, wplus=wplus, gplus=gplus, Fplus=out[0], gdelta=out[1],
                dd=out[2], Gplus=out[3], margin=out[4], accepted=bool(out[5]),
                newton=int(out[6]), ww=out[7])


def ipiano_run(f, filters, theta, l1, l2, cfg: OrcCfg):
    """Algorithm C-0 on one image; returns dict(w, u, trace, iters, trials, status)."""
    f = np.ascontiguousarray(f, np.float32)
    H, W = f.shape
    k, th = _d(filters), _d(theta)
    w = np.empty((H, W))
    trace = np.zeros((cfg.max_iters + 1, TR_FIELDS))
    it, tt = C.c_int(), C.c_int()
    st = lib().orc_ipiano_run(_ptr(f, C.c_float), H, W, _ptr(k), _ptr(th), k.shape[0],
                              k.shape[1], float(l1), float(l2), C.byref(cfg), _ptr(w), _ptr(trace),
                              C.byref(it), C.byref(tt))
    return dict(w=w, u=np.exp(w), trace=trace[: it.value + 1], iters=it.value, trials=tt.value,
                status=st)


def estimate_lipschitz(f, filters, theta, v0, iters=25):
    """rho_hat = |Rayleigh quotient| after ``iters`` power steps on Hess F(w^0) (R-10).

    Returns (rho_hat, L_init = 2^ceil(log2 rho_hat))."""
    f = np.ascontiguousarray(f, np.float32)
    H, W = f.shape
    k, th, v0 = _d(filters), _d(theta), _d(v0)
    Lp = C.c_double()
    rho_hat = lib().orc_estimate_lipschitz(_ptr(f, C.c_float), H, W, _ptr(k), _ptr(th),
                                           k.shape[0], k.shape[1], _ptr(v0), int(iters),
                                           C.byref(Lp))
    return rho_hat, Lp.value


# ------------------------------------------------- variant model (6) in u (f2, I-divergence)

def idiv_energy(u, ft, lam) -> float:
    """D(u,f) = (lam/2) <u^2 - 2 f^2 log u, 1> (Eq.(5))."""
    u, ft = _d(u), _d(ft)
    return float(lib().orc_idiv_energy(_ptr(u), _ptr(ft), u.shape[0], u.shape[1], float(lam)))


def idiv_prox_pixel(uhat, ft, tau, lam) -> float:
    """Closed-form prox of tau D."""
    return float(lib().orc_idiv_prox_pixel(float(uhat), float(ft), float(tau), float(lam)))


def hvp_u(u, v, filters, theta) -> np.ndarray:
    """Hess F(u) v = sum_i theta_i K_i^T [rho''(K_i u) (.) K_i v]."""
    u, v, k, th = _d(u), _d(v), _d(filters), _d(theta)
    out = np.empty_like(u)
    lib().orc_hvp_u(_ptr(u), _ptr(v), u.shape[0], u.shape[1], _ptr(k), _ptr(th), k.shape[0], k.shape[1],
                    _ptr(out))
    return out


def ipiano_trial_u(u, uprev, g, F, L, f, filters, theta, lam, cfg: OrcCfg):
    """One iPiano trial of model (6) in u."""
    u, uprev, g = _d(u), _d(uprev), _d(g)
    ft = ftilde(f)
    k, th = _d(filters), _d(theta)
    uhat, uplus, gplus, out = np.empty_like(u), np.empty_like(u), np.empty_like(u), np.empty(8)
    lib().orc_ipiano_trial_u(_ptr(u), _ptr(uprev), _ptr(g), float(F), float(L), _ptr(ft), u.shape[0],
                             u.shape[1], _ptr(k), _ptr(th), k.shape[0], k.shape[1], float(lam), C.byref(cfg),
                             _ptr(uhat), _ptr(uplus), _ptr(gplus), _ptr(out))
    return dict(uhat=uhat, uplus=uplus, gplus=gplus, Fplus=out[0], gdelta=out[1], dd=out[2], Gplus=out[3],
                margin=out[4], accepted=bool(out[5]), uu=out[7])


def ipiano_run_u(f, filters, theta, lam, cfg: OrcCfg):
    """Model (6) on one image; returns dict(u, trace, iters, trials, status)."""
    f = np.ascontiguousarray(f, np.float32)
    H, W = f.shape
    k, th = _d(filters), _d(theta)
    u = np.empty((H, W))
    trace = np.zeros((cfg.max_iters + 1, TR_FIELDS))
    it, tt = C.c_int(), C.c_int()
    st = lib().orc_ipiano_run_u(_ptr(f, C.c_float), H, W, _ptr(k), _ptr(th), k.shape[0], k.shape[1],
                                float(lam), C.byref(cfg), _ptr(u), _ptr(trace), C.byref(it), C.byref(tt))
    return dict(u=u, trace=trace[: it.value + 1], iters=it.value, trials=tt.value, status=st)


def estimate_lipschitz_u(f, filters, theta, v0, iters=25):
    """Model (6): |Rayleigh quotient| of Hess F(u^0), u^0 = f~; (rho_hat, 2^ceil(log2 rho_hat))."""
    f = np.ascontiguousarray(f, np.float32)
    H, W = f.shape
    k, th, v0 = _d(filters), _d(theta), _d(v0)
    Lp = C.c_double()
    rho_hat = lib().orc_estimate_lipschitz_u(_ptr(f, C.c_float), H, W, _ptr(k), _ptr(th), k.shape[0],
                                             k.shape[1], _ptr(v0), int(iters), C.byref(Lp))
    return rho_hat, Lp.value


def psnr(x, ref, peak=255.0) -> float:
    """10 log10(peak^2 / MSE)."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    mse = np.mean((x - ref) ** 2)
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)
