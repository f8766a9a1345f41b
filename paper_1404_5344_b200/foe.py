"""Thin Python binding of libfoe (include/foe.h) -- argument marshalling only.

Every entry point has the C name and forwards to the CUDA library; no step of the
method is computed here.  Device arrays are torch CUDA tensors (PyTorch provides
device memory and streams only); host arrays are numpy.  There is no CPU fallback:
if libfoe.so cannot be loaded or no sm_100 device is present, calls raise FoeError.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib

FOE_OK = 0
STATUS_NAMES = {
    0: "FOE_OK", 1: "FOE_ERR_INVALID_ARGUMENT", 2: "FOE_ERR_CUDA", 3: "FOE_ERR_OUT_OF_MEMORY",
    4: "FOE_ERR_NONFINITE", 5: "FOE_ERR_BACKTRACK_LIMIT", 6: "FOE_ERR_PROX_NO_CONVERGENCE",
    7: "FOE_ERR_DOMAIN", 8: "FOE_ERR_COMM", 9: "FOE_ERR_UNSUPPORTED",
}
FOE_DATA_COMBINED, FOE_DATA_NAKAGAMI, FOE_DATA_IDIV = 0, 1, 2
FOE_STENCIL_AUTO, FOE_STENCIL_FFMA, FOE_STENCIL_TENSOR = 0, 1, 2
FOE_SOLVER_AUTO, FOE_SOLVER_GRAPH, FOE_SOLVER_PERSISTENT = 0, 1, 2
TRACE_FIELDS = ("F", "G", "H", "L", "trials", "margin", "newton", "relchg")

EXPORTED = (
    "foe_last_error", "foe_status_string", "foe_version", "foe_kernel_launches", "foe_model_create", "foe_model_destroy",
    "foe_energy_grad", "foe_hvp", "foe_estimate_lipschitz", "ipiano_config_default",
    "ipiano_state_create", "ipiano_state_reset", "ipiano_step", "ipiano_solve", "ipiano_get_iterate",
    "ipiano_get_counters", "ipiano_get_trace", "ipiano_profile", "ipiano_profile_read", "ipiano_profile_read_k2",
    "ipiano_state_destroy", "ipiano_state_stencil", "ipiano_state_tiling", "ipiano_state_solver", "ipiano_run",
    "foe_model_set_stencil", "foe_slab_exchange_plan", "foe_comm_unique_id", "foe_comm_create", "foe_comm_init", "foe_comm_destroy", "ipiano_slabs_create", "ipiano_slabs_reset",
    "ipiano_slabs_solve", "ipiano_slabs_advance", "ipiano_slabs_get_iterate", "ipiano_slabs_member", "ipiano_slabs_destroy",
    "ipiano_slabs_halo_handle", "ipiano_slabs_connect_peers", "ipiano_slabs_disconnect_peers",
    "foe_psnr", "foe_ssim", "foe_add_speckle",
)


class FoeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


class IPianoConfig(C.Structure):
    _fields_ = [
        ("beta", C.c_double), ("step_safety", C.c_double), ("backtrack_factor", C.c_double),
        ("shrink", C.c_double), ("max_iters", C.c_int), ("max_backtracks", C.c_int),
        ("newton_max_iters", C.c_int), ("newton_tol", C.c_double), ("rel_change_tol", C.c_double),
        ("w_guard", C.c_double), ("record_trace", C.c_int), ("filter_groups", C.c_int),
        ("stencil", C.c_int), ("solver", C.c_int), ("tile_rows", C.c_int),
    ]


_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)
_configured = None


def lib():
    """The loaded libfoe with argtypes set (raises if it cannot be built/loaded)."""
    global _configured
    if _configured is not None:
        return _configured
    L = _lib.load()
    L.foe_last_error.restype = C.c_char_p
    L.foe_status_string.restype = C.c_char_p
    L.foe_status_string.argtypes = [C.c_int]
    L.foe_version.restype = C.c_char_p
    L.foe_kernel_launches.restype = C.c_longlong
    L.foe_kernel_launches.argtypes = []
    L.foe_model_create.argtypes = [_vp, C.c_int, C.c_int, _vp, _dp, C.c_double, C.c_int, C.c_int,
                                   C.POINTER(_vp)]
    L.foe_model_destroy.argtypes = [_vp]
    L.foe_model_destroy.restype = None
    L.foe_energy_grad.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _vp, _vp]
    L.foe_hvp.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp]
    L.foe_estimate_lipschitz.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int, _dp, _dp, _vp]
    L.ipiano_config_default.argtypes = [C.POINTER(IPianoConfig)]
    L.ipiano_config_default.restype = None
    L.ipiano_state_create.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp,
                                      C.POINTER(IPianoConfig), _vp, C.POINTER(_vp)]
    L.ipiano_state_reset.argtypes = [_vp, _vp, _dp, _vp]
    L.ipiano_step.argtypes = [_vp, _vp, _ip]
    L.ipiano_solve.argtypes = [_vp, _vp]
    L.ipiano_get_iterate.argtypes = [_vp, _vp, _vp, _vp]
    L.ipiano_get_counters.argtypes = [_vp, _ip, _ip, _ip, _dp]
    L.ipiano_get_trace.argtypes = [_vp, _vp, C.c_size_t]
    L.ipiano_profile.argtypes = [_vp, C.c_int]
    L.ipiano_profile_read.argtypes = [_vp, _dp, _llp, _llp]
    L.ipiano_profile_read_k2.argtypes = [_vp, _dp, _llp]
    L.ipiano_state_stencil.argtypes = [_vp]
    L.ipiano_state_stencil.restype = C.c_int
    L.ipiano_state_tiling.argtypes = [_vp, _ip, _ip, _ip]
    L.ipiano_state_solver.argtypes = [_vp]
    L.ipiano_state_solver.restype = C.c_int
    L.ipiano_state_destroy.argtypes = [_vp]
    L.ipiano_state_destroy.restype = None
    L.ipiano_run.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.POINTER(IPianoConfig),
                             _vp, _vp, C.c_size_t, _vp]
    L.foe_model_set_stencil.argtypes = [_vp, C.c_int]
    L.foe_comm_unique_id.argtypes = [_vp]
    L.foe_slab_exchange_plan.argtypes = [C.c_int, C.c_int, _vp]
    L.foe_comm_create.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    L.foe_comm_init.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_vp)]
    L.foe_comm_destroy.argtypes = [_vp]
    L.foe_comm_destroy.restype = None
    L.ipiano_slabs_create.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, _dp, C.c_double,
                                      C.POINTER(IPianoConfig), _vp, _vp, C.POINTER(_vp)]
    L.ipiano_slabs_reset.argtypes = [_vp, _vp, C.c_double, _vp]
    L.ipiano_slabs_solve.argtypes = [_vp, _vp]
    L.ipiano_slabs_advance.argtypes = [_vp, C.c_int, _vp]
    L.ipiano_slabs_get_iterate.argtypes = [_vp, _vp, _vp, _vp]
    L.ipiano_slabs_member.argtypes = [_vp, C.c_int, C.POINTER(_vp)]
    L.ipiano_slabs_halo_handle.argtypes = [_vp, _vp]
    L.ipiano_slabs_connect_peers.argtypes = [_vp, _vp, _vp]
    L.ipiano_slabs_disconnect_peers.argtypes = [_vp]
    L.foe_psnr.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _vp]
    L.foe_ssim.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _vp]
    L.foe_add_speckle.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _dp, C.c_ulonglong, _vp, _vp]
    L.ipiano_slabs_destroy.argtypes = [_vp]
    L.ipiano_slabs_destroy.restype = None
    _configured = L
    return L


def _check(status: int):
    if status != FOE_OK:
        raise FoeError(status, lib().foe_last_error().decode())


def foe_version() -> str:
    return lib().foe_version().decode()


def foe_kernel_launches() -> int:
    """Kernels launched by libfoe in this process (graph replays count each kernel)."""
    return int(lib().foe_kernel_launches())


def foe_last_error() -> str:
    return lib().foe_last_error().decode()


def foe_status_string(status: int) -> str:
    return lib().foe_status_string(int(status)).decode()


# ------------------------------------------------------------------------ marshalling

def _torch():
    import torch
    return torch


def _dev_ptr(t, dtype, name, shape=None, device=None):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the model on cuda:{device}")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        return C.c_void_p(_torch().cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _bhw(t):
    if t.dim() == 2:
        return 1, int(t.shape[0]), int(t.shape[1])
    if t.dim() != 3:
        raise ValueError("images must be [B][H][W] or [H][W]")
    return int(t.shape[0]), int(t.shape[1]), int(t.shape[2])


def _host_d(a, n, name):
    if a is None:
        return None, None
    arr = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    if arr.size != n:
        raise ValueError(f"{name} must have {n} values, got {arr.size}")
    return arr, arr.ctypes.data_as(_dp)


# -------------------------------------------------------------------------- model

class Model:
    """foe_model handle: the FoE bank {(k_i, theta_i)} (Eq.(2)) plus lambda of Eq.(10)."""

    def __init__(self, handle: C.c_void_p, n_filters: int, m: int, device: int):
        self._h = handle
        self.n_filters, self.m, self.device = n_filters, m, device

    @property
    def handle(self):
        if self._h is None:
            raise FoeError(1, "model destroyed")
        return self._h

    def destroy(self):
        if self._h is not None:
            lib().foe_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def foe_model_create(filters, alphas, lam: Optional[Sequence[float]] = None, looks: float = 0.0,
                     term: int = FOE_DATA_COMBINED, device: int = 0) -> Model:
    k = np.ascontiguousarray(np.asarray(filters, np.float32))
    if k.ndim != 3 or k.shape[1] != k.shape[2]:
        raise ValueError("filters must be [n_filters][m][m]")
    a = np.ascontiguousarray(np.asarray(alphas, np.float32).reshape(-1))
    if a.size != k.shape[0]:
        raise ValueError("alphas must have n_filters values")
    lam_arr, lam_p = _host_d(lam, 2, "lam") if lam is not None else (None, None)
    h = C.c_void_p()
    _check(lib().foe_model_create(k.ctypes.data_as(_vp), k.shape[0], k.shape[1], a.ctypes.data_as(_vp),
                                  lam_p, float(looks), int(term), int(device), C.byref(h)))
    return Model(h, k.shape[0], k.shape[1], device)


def foe_model_destroy(model: Model):
    model.destroy()


def foe_model_set_stencil(model: Model, stencil: int):
    """FOE_STENCIL_AUTO / _FFMA (K1) / _TENSOR (K8) for foe_energy_grad with this model."""
    _check(lib().foe_model_set_stencil(model.handle, int(stencil)))


# ----------------------------------------------------------------- energy/gradient

def foe_energy_grad(model: Model, w, f=None, lam_per_image=None, prior=True, data=False, grad=True,
                    stream=None):
    """F(w), G(w) (host fp64 [B]) and grad_w F (device fp32 [B][H][W]) at device fp64 w."""
    torch = _torch()
    B, H, W = _bhw(w)
    wp = _dev_ptr(w, torch.float64, "w", device=model.device)
    fp = _dev_ptr(f, torch.float32, "f", w.shape, model.device) if f is not None else None
    if data and f is None:
        raise ValueError("data energy needs f")
    lam_arr, lam_p = _host_d(lam_per_image, 2 * B, "lam_per_image")
    Fh = np.zeros(B) if prior else None
    Gh = np.zeros(B) if data else None
    g = torch.empty(w.shape, dtype=torch.float32, device=w.device) if grad else None
    _check(lib().foe_energy_grad(model.handle, wp, fp, B, H, W, lam_p,
                                 Fh.ctypes.data_as(_dp) if prior else None,
                                 Gh.ctypes.data_as(_dp) if data else None,
                                 C.c_void_p(g.data_ptr()) if grad else None, _stream(stream)))
    return Fh, Gh, g


def foe_hvp(model: Model, w, v, stream=None):
    torch = _torch()
    B, H, W = _bhw(w)
    hv = torch.empty(w.shape, dtype=torch.float32, device=w.device)
    _check(lib().foe_hvp(model.handle, _dev_ptr(w, torch.float64, "w", device=model.device),
                         _dev_ptr(v, torch.float64, "v", w.shape, model.device), B, H, W,
                         C.c_void_p(hv.data_ptr()), _stream(stream)))
    return hv


def foe_estimate_lipschitz(model: Model, f, v0, power_iters: int = 25, stream=None):
    """(rho_hat [B], L_init [B] = 2^ceil(log2 rho_hat)) -- DESIGN.md R-10."""
    torch = _torch()
    B, H, W = _bhw(f)
    rho = np.zeros(B)
    L = np.zeros(B)
    _check(lib().foe_estimate_lipschitz(model.handle, _dev_ptr(f, torch.float32, "f", device=model.device),
                                        B, H, W, _dev_ptr(v0, torch.float64, "v0", f.shape, model.device),
                                        int(power_iters), rho.ctypes.data_as(_dp), L.ctypes.data_as(_dp),
                                        _stream(stream)))
    return rho, L


# ---------------------------------------------------------------------------- iPiano

def ipiano_config_default(**overrides) -> IPianoConfig:
    cfg = IPianoConfig()
    lib().ipiano_config_default(C.byref(cfg))
    for k, v in overrides.items():
        if not hasattr(cfg, k):
            raise AttributeError(f"ipiano_config has no field {k}")
        setattr(cfg, k, v)
    return cfg


class State:
    """ipiano_state handle: a batch of B independent iPiano problems on one device."""

    def __init__(self, handle, model: Model, B, H, W, cfg: IPianoConfig):
        self._h = handle
        self.model, self.B, self.H, self.W, self.cfg = model, B, H, W, cfg

    @property
    def handle(self):
        if self._h is None:
            raise FoeError(1, "state destroyed")
        return self._h

    def destroy(self):
        if self._h is not None:
            lib().ipiano_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def ipiano_state_create(model: Model, f, lam_per_image=None, lipschitz_init=None,
                        cfg: Optional[IPianoConfig] = None, stream=None) -> State:
    torch = _torch()
    B, H, W = _bhw(f)
    cfg = cfg if cfg is not None else ipiano_config_default()
    lam_arr, lam_p = _host_d(lam_per_image, 2 * B, "lam_per_image")
    L_arr, L_p = _host_d(lipschitz_init, B, "lipschitz_init")
    if L_p is None:
        raise ValueError("lipschitz_init is required (see foe_estimate_lipschitz)")
    h = C.c_void_p()
    _check(lib().ipiano_state_create(model.handle, _dev_ptr(f, torch.float32, "f", device=model.device),
                                     B, H, W, lam_p, L_p, C.byref(cfg), _stream(stream), C.byref(h)))
    return State(h, model, B, H, W, cfg)


def ipiano_state_reset(state: State, f, lipschitz_init, stream=None):
    """Re-initialise ``state`` from new device observations f (same shape), no reallocation."""
    torch = _torch()
    L_arr, L_p = _host_d(lipschitz_init, state.B, "lipschitz_init")
    _check(lib().ipiano_state_reset(state.handle, _dev_ptr(f, torch.float32, "f", (state.B, state.H, state.W),
                                                           state.model.device), L_p, _stream(stream)))


def ipiano_step(state: State, stream=None) -> np.ndarray:
    it = np.zeros(state.B, np.int32)
    _check(lib().ipiano_step(state.handle, _stream(stream), it.ctypes.data_as(_ip)))
    return it


def ipiano_solve(state: State, stream=None):
    _check(lib().ipiano_solve(state.handle, _stream(stream)))


def ipiano_get_iterate(state: State, want_w=True, want_u=True, stream=None, w_out=None, u_out=None):
    """Current iterate: (w fp64, u = e^w fp32) device tensors (preallocated outputs optional)."""
    torch = _torch()
    dev = torch.device("cuda", state.model.device)
    shp = (state.B, state.H, state.W)
    w = w_out if w_out is not None else (torch.empty(shp, dtype=torch.float64, device=dev) if want_w else None)
    u = u_out if u_out is not None else (torch.empty(shp, dtype=torch.float32, device=dev) if want_u else None)
    want_w, want_u = w is not None, u is not None
    if want_w:
        _dev_ptr(w, torch.float64, "w_out", shp, state.model.device)
    if want_u:
        _dev_ptr(u, torch.float32, "u_out", shp, state.model.device)
    _check(lib().ipiano_get_iterate(state.handle, C.c_void_p(w.data_ptr()) if want_w else None,
                                    C.c_void_p(u.data_ptr()) if want_u else None, _stream(stream)))
    return w, u


def ipiano_get_counters(state: State):
    B = state.B
    it = np.zeros(B, np.int32); tr = np.zeros(B, np.int32); stt = np.zeros(B, np.int32); L = np.zeros(B)
    _check(lib().ipiano_get_counters(state.handle, it.ctypes.data_as(_ip), tr.ctypes.data_as(_ip),
                                     stt.ctypes.data_as(_ip), L.ctypes.data_as(_dp)))
    return dict(iters=it, trials=tr, status=stt, L=L)


def ipiano_get_trace(state: State) -> np.ndarray:
    """[B][max_iters+1][8] records (TRACE_FIELDS)."""
    tr = np.zeros((state.B, state.cfg.max_iters + 1, 8))
    _check(lib().ipiano_get_trace(state.handle, tr.ctypes.data_as(_vp), tr.nbytes))
    return tr


def ipiano_profile(state: State, enable: bool = True):
    _check(lib().ipiano_profile(state.handle, int(bool(enable))))


def ipiano_profile_read(state: State):
    ms = C.c_double(); n = C.c_longlong(); tot = C.c_longlong()
    _check(lib().ipiano_profile_read(state.handle, C.byref(ms), C.byref(n), C.byref(tot)))
    return ms.value, n.value, tot.value


def ipiano_profile_read_k2(state: State):
    """(ms, launches) of K2 in the profiled rounds since the last call (graph driver)."""
    ms = C.c_double(); n = C.c_longlong()
    _check(lib().ipiano_profile_read_k2(state.handle, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def ipiano_state_tiling(state: State):
    """(tile_rows, tile_cols, halo_mode) of the state's tensor-core stencil (zeros for FFMA)."""
    r, c, m = C.c_int(), C.c_int(), C.c_int()
    _check(lib().ipiano_state_tiling(state.handle, C.byref(r), C.byref(c), C.byref(m)))
    return r.value, c.value, m.value


def ipiano_state_stencil(state: State) -> int:
    """FOE_STENCIL_FFMA (K1) or FOE_STENCIL_TENSOR (K8): the prior kernel this state runs."""
    return int(lib().ipiano_state_stencil(state.handle))


def ipiano_state_solver(state: State) -> int:
    """FOE_SOLVER_GRAPH or FOE_SOLVER_PERSISTENT: the trial-loop driver this state runs."""
    return int(lib().ipiano_state_solver(state.handle))


def ipiano_state_destroy(state: State):
    state.destroy()


def ipiano_run(model: Model, f, lam_per_image=None, lipschitz_init=None, cfg: Optional[IPianoConfig] = None,
               u_out=None, want_trace=True, stream=None):
    """One-shot solve.  ``f`` and ``u_out`` may be numpy (host) or CUDA tensors (device).

    Returns (u, trace) with u of the same kind as ``u_out`` (allocated like ``f`` if None)."""
    torch = _torch()
    cfg = cfg if cfg is not None else ipiano_config_default()
    if isinstance(f, np.ndarray):
        fh = np.ascontiguousarray(f, np.float32)
        if fh.ndim == 2:
            fh = fh[None]
        B, H, W = fh.shape
        f_ptr = fh.ctypes.data_as(_vp)
        keep = fh
    else:
        B, H, W = _bhw(f)
        f_ptr = _dev_ptr(f, torch.float32, "f", device=model.device)
        keep = f
    if u_out is None:
        u_out = np.empty((B, H, W), np.float32) if isinstance(f, np.ndarray) else torch.empty(
            (B, H, W), dtype=torch.float32, device=f.device)
    if isinstance(u_out, np.ndarray):
        if u_out.dtype != np.float32 or not u_out.flags.c_contiguous or u_out.size != B * H * W:
            raise ValueError("u_out must be a contiguous float32 array of B*H*W values")
        u_ptr = u_out.ctypes.data_as(_vp)
    else:
        u_ptr = _dev_ptr(u_out, torch.float32, "u_out", device=model.device)
    lam_arr, lam_p = _host_d(lam_per_image, 2 * B, "lam_per_image")
    L_arr, L_p = _host_d(lipschitz_init, B, "lipschitz_init")
    if L_p is None:
        raise ValueError("lipschitz_init is required")
    trace = np.zeros((B, cfg.max_iters + 1, 8)) if want_trace else None
    _check(lib().ipiano_run(model.handle, f_ptr, B, H, W, lam_p, L_p, C.byref(cfg), u_ptr,
                            trace.ctypes.data_as(_vp) if want_trace else None,
                            trace.nbytes if want_trace else 0, _stream(stream)))
    del keep
    return u_out, trace


# ------------------------------------------------------------------ row slabs (multi-GPU)

class Comm:
    """foe_comm handle: this rank's NCCL communicator for the row-slab halo exchange."""

    def __init__(self, handle, nranks: int, rank: int, device: int):
        self._h = handle
        self.nranks, self.rank, self.device = nranks, rank, device

    @property
    def handle(self):
        if self._h is None:
            raise FoeError(1, "comm destroyed")
        return self._h

    def destroy(self):
        if self._h is not None:
            lib().foe_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


FOE_HALO_SEND, FOE_HALO_RECV = 0, 1
FOE_HALO_TOP_ROWS, FOE_HALO_BOTTOM_GHOST, FOE_HALO_BOTTOM_ROWS, FOE_HALO_TOP_GHOST = 0, 1, 2, 3


def foe_slab_exchange_plan(nranks: int, rank: int):
    """The ghost-row exchange the library posts on rank `rank` (include/foe.h): four
    (op, peer, buffer) triples in posting order.  Host only: no GPU needed."""
    plan = (C.c_int * 12)()
    _check(lib().foe_slab_exchange_plan(int(nranks), int(rank), C.cast(plan, _vp)))
    return [tuple(plan[3 * k: 3 * k + 3]) for k in range(4)]


def foe_comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().foe_comm_unique_id(C.cast(buf, _vp)))
    return buf.raw


def foe_comm_create(unique_id: bytes, nranks: int, rank: int, device: int) -> Comm:
    if len(unique_id) != 128:
        raise ValueError("unique_id must be the 128 bytes of foe_comm_unique_id")
    buf = C.create_string_buffer(bytes(unique_id), 128)
    h = C.c_void_p()
    _check(lib().foe_comm_create(C.cast(buf, _vp), int(nranks), int(rank), int(device), C.byref(h)))
    return Comm(h, nranks, rank, device)


def foe_comm_init(unique_id: bytes, nranks: int, rank: int) -> Comm:
    """SURVEY.md 8(b)'s name: foe_comm_create on the current CUDA device."""
    import torch
    return foe_comm_create(unique_id, nranks, rank, torch.cuda.current_device())


def foe_comm_destroy(comm: Comm):
    comm.destroy()


class Slabs:
    """ipiano_slabs handle: one scene cut into row slabs (all in-process, or this rank's)."""

    def __init__(self, handle, model: Model, rows: int, W: int, H_global: int, nmembers: int,
                 cfg: IPianoConfig, comm: Optional[Comm]):
        self._h = handle
        self.model, self.rows, self.W, self.H_global = model, rows, W, H_global
        self.nmembers, self.cfg, self.comm = nmembers, cfg, comm

    @property
    def handle(self):
        if self._h is None:
            raise FoeError(1, "slabs destroyed")
        return self._h

    def destroy(self):
        if self._h is not None:
            lib().ipiano_slabs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def ipiano_slabs_create(model: Model, f, H_global: int, nslabs: int = 1, lam=None, lipschitz_init=None,
                        cfg: Optional[IPianoConfig] = None, comm: Optional[Comm] = None, stream=None) -> Slabs:
    """Row-slab decomposition of one H_global x W scene.  comm=None: ``f`` is the whole scene
    [H_global][W] and all ``nslabs`` slabs run in this process; else ``f`` is this rank's slab."""
    torch = _torch()
    if f.dim() != 2:
        raise ValueError("f must be [rows][W]")
    rows, W = int(f.shape[0]), int(f.shape[1])
    cfg = cfg if cfg is not None else ipiano_config_default()
    lam_arr, lam_p = _host_d(lam, 2, "lam")
    if lipschitz_init is None:
        raise ValueError("lipschitz_init is required (see foe_estimate_lipschitz)")
    h = C.c_void_p()
    _check(lib().ipiano_slabs_create(model.handle, _dev_ptr(f, torch.float32, "f", device=model.device),
                                     int(H_global), W, int(nslabs), lam_p, float(lipschitz_init), C.byref(cfg),
                                     comm.handle if comm is not None else None, _stream(stream), C.byref(h)))
    return Slabs(h, model, rows, W, int(H_global), 1 if comm is not None else int(nslabs), cfg, comm)


def ipiano_slabs_reset(slabs: Slabs, f, lipschitz_init: float, stream=None):
    torch = _torch()
    _check(lib().ipiano_slabs_reset(slabs.handle, _dev_ptr(f, torch.float32, "f", (slabs.rows, slabs.W),
                                                           slabs.model.device), float(lipschitz_init),
                                    _stream(stream)))


def ipiano_slabs_solve(slabs: Slabs, stream=None):
    _check(lib().ipiano_slabs_solve(slabs.handle, _stream(stream)))


def ipiano_slabs_advance(slabs: Slabs, target_iters: int, stream=None):
    """Run accepted iterations until min(target_iters, max_iters) are done (include/foe.h)."""
    _check(lib().ipiano_slabs_advance(slabs.handle, int(target_iters), _stream(stream)))


def ipiano_slabs_get_iterate(slabs: Slabs, want_w=True, want_u=True, stream=None, u_out=None):
    """(w fp64, u fp32) device tensors [rows][W] of the slabs owned by this process."""
    torch = _torch()
    dev = torch.device("cuda", slabs.model.device)
    shp = (slabs.rows, slabs.W)
    w = torch.empty(shp, dtype=torch.float64, device=dev) if want_w else None
    u = u_out if u_out is not None else (torch.empty(shp, dtype=torch.float32, device=dev) if want_u else None)
    if u is not None:
        _dev_ptr(u, torch.float32, "u_out", shp, slabs.model.device)
    _check(lib().ipiano_slabs_get_iterate(slabs.handle, C.c_void_p(w.data_ptr()) if w is not None else None,
                                          C.c_void_p(u.data_ptr()) if u is not None else None, _stream(stream)))
    return w, u


def ipiano_slabs_member(slabs: Slabs, j: int = 0) -> State:
    """Non-owning State view of slab member j (counters, trace, profiling)."""
    h = C.c_void_p()
    _check(lib().ipiano_slabs_member(slabs.handle, int(j), C.byref(h)))
    st = State(h, slabs.model, 1, slabs.rows // slabs.nmembers, slabs.W, slabs.cfg)
    st._h_borrowed = h
    st.destroy = lambda: None   # owned by the Slabs handle
    return st


def ipiano_slabs_destroy(slabs: Slabs):
    slabs.destroy()


def ipiano_slabs_halo_handle(slabs: Slabs) -> bytes:
    """This rank's ghost-row buffer as a CUDA IPC handle (64 bytes) for its ring neighbours."""
    buf = C.create_string_buffer(64)
    _check(lib().ipiano_slabs_halo_handle(slabs.handle, C.cast(buf, _vp)))
    return buf.raw


def ipiano_slabs_connect_peers(slabs: Slabs, up_handle: bytes, down_handle: bytes):
    """Switch the ghost-row exchange to direct NVLink stores from K2 (see include/foe.h)."""
    ub = C.create_string_buffer(bytes(up_handle), 64)
    db = C.create_string_buffer(bytes(down_handle), 64)
    _check(lib().ipiano_slabs_connect_peers(slabs.handle, C.cast(ub, _vp), C.cast(db, _vp)))


def ipiano_slabs_disconnect_peers(slabs: Slabs):
    """Back to the ncclSend/Recv exchange (all ranks must take the same path)."""
    _check(lib().ipiano_slabs_disconnect_peers(slabs.handle))


# ------------------------------------------------- evaluation and synthesis

def foe_psnr(x, ref, peak: float = 255.0, stream=None) -> np.ndarray:
    """PSNR per image of device fp32 [B][H][W] tensors (host fp64 [B])."""
    torch = _torch()
    B, H, W = _bhw(x)
    out = np.zeros(B)
    _check(lib().foe_psnr(_dev_ptr(x, torch.float32, "x"), _dev_ptr(ref, torch.float32, "ref", x.shape), B, H, W,
                          float(peak), out.ctypes.data_as(_dp), _stream(stream)))
    return out


def foe_ssim(x, ref, peak: float = 255.0, stream=None) -> np.ndarray:
    """Mean SSIM per image (11x11 Gaussian window, valid region)."""
    torch = _torch()
    B, H, W = _bhw(x)
    out = np.zeros(B)
    _check(lib().foe_ssim(_dev_ptr(x, torch.float32, "x"), _dev_ptr(ref, torch.float32, "ref", x.shape), B, H, W,
                          float(peak), out.ctypes.data_as(_dp), _stream(stream)))
    return out


def foe_add_speckle(u, looks, seed: int, stream=None):
    """f = u sqrt(s), s ~ Gamma(L, 1/L) per image, Philox4x32-10 counter-based (device fp32)."""
    torch = _torch()
    B, H, W = _bhw(u)
    lk, lp = _host_d(np.broadcast_to(np.asarray(looks, np.float64), (B,)), B, "looks")
    f = torch.empty_like(u)
    _check(lib().foe_add_speckle(_dev_ptr(u, torch.float32, "u"), B, H, W, lp, C.c_ulonglong(int(seed)),
                                 C.c_void_p(f.data_ptr()), _stream(stream)))
    return f
