"""Thin ctypes binding of the C ABI in include/lfm.h (argument marshalling only).

Every step of the hot path runs inside liblfm.so (hand-written sm_100a kernels).  Device arrays are
passed as raw pointers taken from torch CUDA tensors (torch provides device memory, streams and
process groups only); there is no CPU fallback: if the library is missing, importing this module
raises.  Names follow the C ABI one to one.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblfm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2208_11422_b200.build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

LFM_OK, LFM_EINVAL, LFM_EDIM, LFM_ENEG, LFM_EZERO, LFM_ENOMEM, LFM_ECUDA, LFM_ENCCL, LFM_EUNSUPPORTED = range(9)
STATUS_NAMES = ["LFM_OK", "LFM_EINVAL", "LFM_EDIM", "LFM_ENEG", "LFM_EZERO", "LFM_ENOMEM", "LFM_ECUDA", "LFM_ENCCL",
                "LFM_EUNSUPPORTED"]
LFM_MODE_FIXED, LFM_MODE_AUTO = 0, 1
LFM_REGION_TRIANGLE, LFM_REGION_RECTANGLE = 0, 1
LFM_UPDATE_RL, LFM_UPDATE_ISRA = 0, 1
LFM_PLAN_NO_COMM, LFM_PLAN_DIRECT, LFM_PLAN_FFT_ONLY, LFM_PLAN_TC_DIRECT, LFM_PLAN_GRAPHS, LFM_PLAN_NO_TC = 1, 2, 4, 16, 32, 64
LFM_PLAN_DEVICE_LOOP, LFM_PLAN_EVEN_SHARDS, LFM_PLAN_FORCE_COMM, LFM_PLAN_SYMMETRIC = 128, 256, 512, 1024
LFM_PLAN_FRAMES = 2048
LFM_PLAN_TILES, LFM_PLAN_NO_TILES = 4096, 8192


class LfmError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


class lfm_optics(ctypes.Structure):
    _fields_ = [("wavelength_um", ctypes.c_double), ("na", ctypes.c_double),
                ("mla_pitch_um", ctypes.c_double), ("magnification", ctypes.c_double)]


class lfm_policy(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("n_iters", ctypes.c_int), ("max_iters", ctypes.c_int),
                ("min_iters", ctypes.c_int), ("patience", ctypes.c_int), ("eps", ctypes.c_float),
                ("region", ctypes.c_int), ("init_from_x", ctypes.c_int), ("update", ctypes.c_int)]


class lfm_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_id", ctypes.c_ubyte * 128)]


class lfm_info(ctypes.Structure):
    _fields_ = [("nnum", ctypes.c_int), ("nz", ctypes.c_int), ("kh", ctypes.c_int), ("kw", ctypes.c_int),
                ("height", ctypes.c_int), ("width", ctypes.c_int), ("unit_begin", ctypes.c_int),
                ("unit_end", ctypes.c_int), ("fft_h", ctypes.c_int), ("fft_w", ctypes.c_int),
                ("lc_min_h", ctypes.c_int), ("lc_min_w", ctypes.c_int), ("n_kappa", ctypes.c_int),
                ("units_padded", ctypes.c_int), ("x_s", ctypes.c_int), ("y_s", ctypes.c_int),
                ("direct", ctypes.c_int), ("transfer_bytes", ctypes.c_size_t), ("device_bytes", ctypes.c_size_t),
                ("plan_ms", ctypes.c_double), ("direct_planes", ctypes.c_int), ("fft_units", ctypes.c_int),
                ("tc_planes", ctypes.c_int), ("tc_flops_executed", ctypes.c_double), ("tc_flops_algorithmic", ctypes.c_double),
                ("planes_moved_for_memory", ctypes.c_int), ("partition_sms", (ctypes.c_int * 2) * 2),
                ("c1_mode", ctypes.c_int), ("tc_moved_to_fft", ctypes.c_int), ("tiles", ctypes.c_int),
                ("tile_T1", ctypes.c_int), ("tile_T2", ctypes.c_int), ("tile_groups", ctypes.c_int),
                ("fft_bytes", ctypes.c_double)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["partition_sms"] = [[self.partition_sms[i][j] for j in range(2)] for i in range(2)]
        return d


_P = ctypes.c_void_p
_F = ctypes.POINTER(ctypes.c_float)
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_i = ctypes.c_int


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_lib_policy_default = _sig("lfm_policy_default", lfm_policy, [])
_lib_last_error = _sig("lfm_last_error", ctypes.c_char_p, [])
_lib_version = _sig("lfm_version", ctypes.c_char_p, [])
_lib_shard_units = _sig("lfm_shard_units", _i, [_i, _i, _i, _i, _I, _I])
_lib_partition_model = _sig("lfm_partition_model", _i, [ctypes.c_double, ctypes.c_double, _i, _i, ctypes.c_double, _I, _D])
_lib_tile_model = _sig("lfm_tile_model", _i, [_i, _i, _i, _i, _i, _i, _i, _i, _I, _I, _I, _I, _D, _D])
_lib_unique_id = _sig("lfm_comm_unique_id", _i, [ctypes.POINTER(ctypes.c_ubyte)])
_lib_estimate = _sig("lfm_plan_estimate", _i, [_i, _i, _i, _i, _i, _i, _i, _i, ctypes.c_size_t,
                                               ctypes.POINTER(ctypes.c_size_t), ctypes.c_char_p, ctypes.c_size_t])
_lib_create = _sig("lfm_plan_create", _i, [ctypes.POINTER(_P), _P, _P, _i, _i, _i, _i, _i, _i,
                                           ctypes.POINTER(lfm_optics), ctypes.POINTER(lfm_dist), _i, _P])
_lib_info = _sig("lfm_plan_info", _i, [_P, ctypes.POINTER(lfm_info)])
_lib_owned = _sig("lfm_plan_owned", _i, [_P, ctypes.POINTER(_i), ctypes.POINTER(_i)])
_lib_memlimit = _sig("lfm_set_memory_limit", _i, [ctypes.c_size_t])
_lib_shard_bal = _sig("lfm_shard_units_balanced", _i, [_P, _i, _i, _i, _i, _i, _i, _i, _i, _i, ctypes.POINTER(_i),
                                                      ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_double)])
_lib_destroy = _sig("lfm_plan_destroy", None, [_P])
_lib_forward = _sig("lfm_forward", _i, [_P, _P, _P, _P])
_lib_backward = _sig("lfm_backward", _i, [_P, _P, _P, _P])
_lib_normalizer = _sig("lfm_normalizer", _i, [_P, _P, _P])
_lib_rl_step = _sig("lfm_rl_step", _i, [_P, _P, _P, _P, ctypes.c_float, _i, _P, _D, _P])
_lib_rl_iterate = _sig("lfm_rl_iterate", _i, [_P, _P, _P, ctypes.POINTER(lfm_policy), _I, _I, _D, _F, _P])
_lib_deconvolve_host = _sig("lfm_deconvolve_host", _i, [_P, _P, _P, ctypes.POINTER(lfm_policy), _I, _I, _D, _F, _P])
_lib_quality = _sig("lfm_quality", _i, [_P, _P, _i, _D, _P])
_lib_rl_iterate_batch = _sig("lfm_rl_iterate_batch", _i, [_P, _i, _P, _P, ctypes.POINTER(lfm_policy), _I, _I, _D, _F,
                                                          _P])
_lib_dct_entropy = _sig("lfm_dct_entropy", _i, [_P, _i, _i, _i, ctypes.POINTER(lfm_optics), _i, _D, _I, _I, _P])

LFM_N_STAGES = 11


class lfm_profile_t(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * LFM_N_STAGES), ("count", ctypes.c_longlong * LFM_N_STAGES),
                ("launches", ctypes.c_longlong), ("iterations", ctypes.c_longlong),
                ("kern_ms", ctypes.c_double * 4), ("kern_count", ctypes.c_longlong * 4), ("d2h_bytes", ctypes.c_longlong)]

KERNEL_NAMES = ["tc_fwd", "mac_fwd", "tc_bwd", "mac_bwd"]


_lib_profile = _sig("lfm_profile", _i, [_P, _i])
_lib_profile_read = _sig("lfm_profile_read", _i, [_P, ctypes.POINTER(lfm_profile_t), _i])
_lib_stage_name = _sig("lfm_profile_stage_name", ctypes.c_char_p, [_i])
STAGE_NAMES = [_lib_stage_name(i).decode() for i in range(LFM_N_STAGES)]

EXPORTED = ["lfm_partition_model", "lfm_tile_model", "lfm_shard_units", "lfm_policy_default", "lfm_last_error", "lfm_version", "lfm_comm_unique_id", "lfm_plan_estimate",
            "lfm_plan_create", "lfm_plan_info", "lfm_plan_owned", "lfm_set_memory_limit", "lfm_shard_units_balanced", "lfm_plan_destroy", "lfm_forward", "lfm_backward", "lfm_normalizer",
            "lfm_rl_step", "lfm_rl_iterate", "lfm_deconvolve_host", "lfm_quality", "lfm_dct_entropy",
            "lfm_profile", "lfm_profile_read", "lfm_profile_stage_name", "lfm_rl_iterate_batch"]


def _check(st):
    if st != LFM_OK:
        raise LfmError(st, _lib_last_error().decode())


def _ptr(t):
    """Raw pointer of a torch tensor / numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(t.ctypes.data)
    raise TypeError(type(t))


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _check_dev(t, shape, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _check_host(a, shape, name):
    """Host buffers cross the ABI as raw pointers: the library reads / writes prod(shape) float32 values."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
        raise TypeError(f"{name} must be a C-contiguous float32 numpy array")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(a.shape)}, expected {tuple(shape)}")


def lfm_policy_default():
    return _lib_policy_default()


def lfm_version():
    return _lib_version().decode()


def lfm_last_error():
    return _lib_last_error().decode()


def make_optics(wavelength_um, na, mla_pitch_um, magnification):
    return lfm_optics(wavelength_um, na, mla_pitch_um, magnification)


def make_policy(mode="auto", n_iters=10, max_iters=50, min_iters=2, patience=1, eps=1e-6, region="triangle",
                init_from_x=False, update="rl"):
    p = lfm_policy_default()
    p.mode = LFM_MODE_AUTO if mode == "auto" else LFM_MODE_FIXED
    p.n_iters, p.max_iters, p.min_iters, p.patience = n_iters, max_iters, min_iters, patience
    p.eps = eps
    p.region = LFM_REGION_TRIANGLE if region == "triangle" else LFM_REGION_RECTANGLE
    p.init_from_x = 1 if init_from_x else 0
    p.update = LFM_UPDATE_RL if update == "rl" else LFM_UPDATE_ISRA
    return p


def lfm_comm_unique_id():
    buf = (ctypes.c_ubyte * 128)()
    _check(_lib_unique_id(buf))
    return bytes(buf)


def lfm_shard_units_balanced(psf, nnum, height, width, world, rank, flags=0):
    """(unit_begin, unit_end, est_seconds) of `rank` under the cost-balanced sharding (include/lfm.h)."""
    psf = np.ascontiguousarray(psf, dtype=np.float32)
    nz, kh, kw = psf.shape[0], psf.shape[3], psf.shape[4]
    b, e, t = _i(), _i(), ctypes.c_double()
    _check(_lib_shard_bal(psf.ctypes.data, nnum, nz, kh, kw, height, width, world, rank, flags, ctypes.byref(b),
                          ctypes.byref(e), ctypes.byref(t)))
    return b.value, e.value, t.value


def lfm_set_memory_limit(nbytes):
    """Cap the device memory later plans may use (0 = free memory); see include/lfm.h."""
    _check(_lib_memlimit(int(nbytes)))


def lfm_partition_model(t_tc_ms, mac_bytes, direction, num_sms=148, mac_rate_scale=1.0):
    """(tensor-core SMs, predicted ms) the planner picks for one projection direction; host-only."""
    sms = ctypes.c_int(0)
    ms = ctypes.c_double(0.0)
    _check(_lib_partition_model(float(t_tc_ms), float(mac_bytes), int(direction), int(num_sms), float(mac_rate_scale),
                                ctypes.byref(sms), ctypes.byref(ms)))
    return sms.value, ms.value


def lfm_tile_model(nnum, height, width, d1a, d1b, d2a, d2b, flags=0):
    """The planner's overlap-save tiling for coarse taps in [d1a, d1b] x [d2a, d2b]: dict with L (0:
    none), T1, T2, ntile, cost_unit, cost_whole (seconds per frequency-path unit and iteration); host-only."""
    v = [ctypes.c_int(0) for _ in range(4)]
    cu, cw = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(_lib_tile_model(int(nnum), int(height), int(width), int(d1a), int(d1b), int(d2a), int(d2b), int(flags),
                           *[ctypes.byref(x) for x in v], ctypes.byref(cu), ctypes.byref(cw)))
    return dict(L=v[0].value, T1=v[1].value, T2=v[2].value, ntile=v[3].value, cost_unit=cu.value, cost_whole=cw.value)


def lfm_shard_units(nz, nnum, world, rank):
    b, e = ctypes.c_int(0), ctypes.c_int(0)
    _check(_lib_shard_units(nz, nnum, world, rank, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def lfm_plan_estimate(nnum, nz, kh, kw, height, width, world=1, flags=0, budget_bytes=0):
    out = ctypes.c_size_t(0)
    term = ctypes.create_string_buffer(256)
    _check(_lib_estimate(nnum, nz, kh, kw, height, width, world, flags, budget_bytes, ctypes.byref(out), term, 256))
    return out.value, term.value.decode()


class Plan:
    """Owns an lfm_plan (C handle).  Methods map one to one to the ABI calls."""

    def __init__(self, psf, nnum, height, width, optics=None, rank=0, world=1, nccl_id=None, flags=0, stream=None,
                 psf_t=None):
        psf = np.ascontiguousarray(psf, dtype=np.float32)
        psf_t = None if psf_t is None else np.ascontiguousarray(psf_t, dtype=np.float32)
        if psf_t is not None and psf_t.shape != psf.shape:
            raise ValueError("psf_t must have the shape of psf")
        if psf.ndim != 5 or psf.shape[1] != nnum or psf.shape[2] != nnum:
            raise ValueError("psf must be [nz][N][N][kh][kw]")
        nz, _, _, kh, kw = psf.shape
        self.nz, self.nnum, self.kh, self.kw, self.height, self.width = nz, nnum, kh, kw, height, width
        dist = None
        if world > 1 or rank or nccl_id is not None:
            dist = lfm_dist()
            dist.rank, dist.world = rank, world
            if nccl_id is not None:
                ctypes.memmove(dist.nccl_id, bytes(nccl_id), 128)
        h = _P()
        opt = optics if (optics is None or isinstance(optics, lfm_optics)) else lfm_optics(*optics)
        _check(_lib_create(ctypes.byref(h), _ptr(psf), _ptr(psf_t), nnum, nz, kh, kw, height, width,
                           ctypes.byref(opt) if opt is not None else None,
                           ctypes.byref(dist) if dist is not None else None, flags, _stream(stream)))
        self._h = h

    # -- lifetime --
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls --
    def info(self):
        inf = lfm_info()
        _check(_lib_info(self._h, ctypes.byref(inf)))
        return inf.as_dict()

    def owned(self):
        """(unit_begin, unit_end) this rank owns (lfm_plan_owned)."""
        b, e = _i(), _i()
        _check(_lib_owned(self._h, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def forward(self, x, y, stream=None):
        _check_dev(x, (self.nz, self.height, self.width), "x")
        _check_dev(y, (self.height, self.width), "y")
        _check(_lib_forward(self._h, _ptr(x), _ptr(y), _stream(stream)))

    def backward(self, y, x, stream=None):
        _check_dev(y, (self.height, self.width), "y")
        _check_dev(x, (self.nz, self.height, self.width), "x")
        _check(_lib_backward(self._h, _ptr(y), _ptr(x), _stream(stream)))

    def normalizer(self, x, stream=None):
        _check_dev(x, (self.nz, self.height, self.width), "x")
        _check(_lib_normalizer(self._h, _ptr(x), _stream(stream)))

    def rl_step(self, y, x_in, x_out, eps=1e-6, region=LFM_REGION_TRIANGLE, yhat_out=None, entropy=True,
                stream=None):
        _check_dev(y, (self.height, self.width), "y")
        _check_dev(x_in, (self.nz, self.height, self.width), "x_in")
        _check_dev(x_out, (self.nz, self.height, self.width), "x_out")
        e = ctypes.c_double(0.0)
        _check(_lib_rl_step(self._h, _ptr(y), _ptr(x_in), _ptr(x_out), eps, region, _ptr(yhat_out),
                            ctypes.byref(e) if entropy else None, _stream(stream)))
        return e.value if entropy else None

    def rl_iterate(self, y, x, policy, want_ms=False, stream=None):
        _check_dev(y, (self.height, self.width), "y")
        _check_dev(x, (self.nz, self.height, self.width), "x")
        cap = max(policy.n_iters, policy.max_iters)
        series = (ctypes.c_double * cap)()
        ms = (ctypes.c_float * cap)() if want_ms else None
        best, stop = ctypes.c_int(0), ctypes.c_int(0)
        _check(_lib_rl_iterate(self._h, _ptr(y), _ptr(x), ctypes.byref(policy), ctypes.byref(best),
                               ctypes.byref(stop), series, ms, _stream(stream)))
        out = dict(best_iter=best.value, stop_iter=stop.value, series=list(series[:stop.value]))
        if want_ms:
            out["ms"] = list(ms[:stop.value])
        return out

    def rl_iterate_batch(self, y, x, policy, want_ms=False, stream=None):
        """Lockstep RL over F frames (y [F,H,W], x [F,nz,H,W] CUDA tensors); per-frame results."""
        F = y.shape[0]
        _check_dev(y, (F, self.height, self.width), "y")
        _check_dev(x, (F, self.nz, self.height, self.width), "x")
        cap = max(policy.n_iters, policy.max_iters)
        series = (ctypes.c_double * (cap * F))()
        ms = (ctypes.c_float * cap)() if want_ms else None
        best, stop = (ctypes.c_int * F)(), (ctypes.c_int * F)()
        _check(_lib_rl_iterate_batch(self._h, F, _ptr(y), _ptr(x), ctypes.byref(policy), best, stop, series, ms,
                                     _stream(stream)))
        out = dict(best_iter=list(best), stop_iter=list(stop),
                   series=[list(series[f * cap:f * cap + stop[f]]) for f in range(F)])
        if want_ms:
            out["ms"] = list(ms[:max(stop)])
        return out

    def deconvolve_host(self, y_host, x_host, policy, want_ms=False, stream=None):
        """End-to-end call with host buffers (numpy float32, ideally pinned torch CPU tensors)."""
        _check_host(y_host, (self.height, self.width), "y_host")
        _check_host(x_host, (self.nz, self.height, self.width), "x_host")
        if not x_host.flags["WRITEABLE"]:
            raise ValueError("x_host must be writeable")
        cap = max(policy.n_iters, policy.max_iters)
        series = (ctypes.c_double * cap)()
        ms = (ctypes.c_float * cap)() if want_ms else None
        best, stop = ctypes.c_int(0), ctypes.c_int(0)
        _check(_lib_deconvolve_host(self._h, _ptr(y_host), _ptr(x_host), ctypes.byref(policy), ctypes.byref(best),
                                    ctypes.byref(stop), series, ms, _stream(stream)))
        out = dict(best_iter=best.value, stop_iter=stop.value, series=list(series[:stop.value]))
        if want_ms:
            out["ms"] = list(ms[:stop.value])
        return out

    def profile(self, enable=True):
        _check(_lib_profile(self._h, 1 if enable else 0))

    def profile_read(self, reset=False):
        """Per-stage summed device ms / counts, kernel launches and iterations since the last reset."""
        pr = lfm_profile_t()
        _check(_lib_profile_read(self._h, ctypes.byref(pr), 1 if reset else 0))
        return dict(ms={STAGE_NAMES[i]: pr.ms[i] for i in range(LFM_N_STAGES)},
                    count={STAGE_NAMES[i]: pr.count[i] for i in range(LFM_N_STAGES)},
                    launches=pr.launches, iterations=pr.iterations,
                    kern_ms={KERNEL_NAMES[i]: pr.kern_ms[i] for i in range(4)},
                    kern_count={KERNEL_NAMES[i]: pr.kern_count[i] for i in range(4)}, d2h_bytes=pr.d2h_bytes)

    def quality(self, x, region=LFM_REGION_TRIANGLE, stream=None):
        _check_dev(x, (self.nz, self.height, self.width), "x")
        e = ctypes.c_double(0.0)
        _check(_lib_quality(self._h, _ptr(x), region, ctypes.byref(e), _stream(stream)))
        return e.value


def lfm_dct_entropy(img, nnum, optics, region=LFM_REGION_TRIANGLE, stream=None):
    H, W = img.shape
    _check_dev(img, (H, W), "img")
    e = ctypes.c_double(0.0)
    xs, ys = ctypes.c_int(0), ctypes.c_int(0)
    opt = optics if isinstance(optics, lfm_optics) else lfm_optics(*optics)
    _check(_lib_dct_entropy(_ptr(img), H, W, nnum, ctypes.byref(opt), region, ctypes.byref(e), ctypes.byref(xs),
                            ctypes.byref(ys), _stream(stream)))
    return e.value, xs.value, ys.value
