"""Batched drop-in for the reference's solver entry points.

Reference boundary (pure Python, /root/reference/pkg/src/ladlasso):
  locus.solve_locus(spec, cfg)              locus.py:300-409
  ccd.ccd_descend(spec, start, cfg)         ccd.py:126-206
  brute.solve_brute(spec, caps)             brute.py:106-145
  model.evaluate_objective(spec, beta)      model.py:151-154
Here each becomes one call over B problems (X (B, n, p), y (B, n), lam (B,)).
Host (numpy) inputs go through the host-buffer C entry point (the copies are
part of the call); CUDA torch tensors stay on the device and run on the
current torch stream.  There is no CPU implementation behind any of these.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import DEFAULT_LAMBDA_FLOOR, CcdConfig, LocusConfig, locus_params
from .errors import (DeviceError, DimensionMismatchError, InvalidInputError, ProblemTooLargeError,
                     UnboundedDirectionError)

STATUS_OK = 0
STATUS_UNBOUNDED = 1
STATUS_INVALID = 2
STATUS_SCRATCH = 3


def _to_device(a, dev):
    """Host array -> device tensor with no host-side copy: lad_copy_h2d issues cudaMemcpyAsync on
    the array's own pointer, so page-locked caller buffers copy by DMA (torch's copy of a numpy
    view does not know the memory is pinned and stages it: ~9 GB/s measured)."""
    import torch

    a = np.ascontiguousarray(a)
    if not a.dtype.isnative:  # the copy moves raw bytes: bring foreign byte order to native first
        a = a.astype(a.dtype.newbyteorder("="))
    t = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), device=dev)
    _check(_lib.load().lad_copy_h2d(t.data_ptr(), a.ctypes.data, a.nbytes, torch.cuda.current_stream(dev).cuda_stream))
    return t


def _to_host(t):
    """Device tensor -> numpy array in page-locked memory (torch's caching host allocator), so the
    result copy is a DMA; a fresh pageable array faults its pages in during the copy (~2 GB/s
    measured for 32 MB of brute-force results)."""
    import torch

    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _host_empty(shape, dtype=np.float64):
    """Uninitialised page-locked numpy array (output buffers of the host-buffer C ABI calls)."""
    import torch

    return torch.empty(shape, dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True).numpy()


def _is_torch(a) -> bool:
    try:
        import torch

        return isinstance(a, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _check(rc: int):
    if rc == _lib.LAD_OK:
        return
    msg = _lib.last_error()
    if rc == _lib.LAD_E_INVALID:
        raise InvalidInputError(msg)
    if rc == _lib.LAD_E_TOO_LARGE:
        raise ProblemTooLargeError(msg)
    if rc == _lib.LAD_E_UNSUPPORTED:
        raise InvalidInputError(msg)
    raise DeviceError(msg)


@dataclass
class BatchedSolveResult:
    """Per-problem SolveResult fields (model.py:113-133) as arrays."""

    beta: object            # (B, p)
    objective: object       # (B,)
    iterations: object      # (B,) int32
    objective_evals: object  # (B,) int32
    converged: object       # (B,) bool
    status: object          # (B,) uint8: 0 ok, 1 unbounded, 2 invalid
    descents: object        # (B,) int32: ccd_descend calls
    steps: object           # (B,) int64: exact coordinate steps
    solver_id: str
    wall_time: float

    def raise_for_status(self):
        st = np.asarray(self.status.cpu() if _is_torch(self.status) else self.status)
        if (st == STATUS_UNBOUNDED).any():
            i = int(np.nonzero(st == STATUS_UNBOUNDED)[0][0])
            raise UnboundedDirectionError(f"problem {i}: no interior minimum found after 60 bracket extensions")
        if (st == STATUS_INVALID).any():
            i = int(np.nonzero(st == STATUS_INVALID)[0][0])
            raise InvalidInputError(f"problem {i}: non-finite data, invalid lambda or invalid bracket")
        if (st == STATUS_SCRATCH).any():
            i = int(np.nonzero(st == STATUS_SCRATCH)[0][0])
            raise DeviceError(f"problem {i}: curve-point scratch exceeded (re-run with a larger seen_capacity)")


def _is_f32(X) -> bool:
    """fp32 mode is selected by a binary32 design matrix (numpy or torch)."""
    dt = getattr(X, "dtype", None)
    if dt is None:
        return False
    if _is_torch(X):
        import torch

        return dt == torch.float32
    return dt == np.float32


def _validate_host(X, y, lam, f32=False):
    ft = np.float32 if f32 else np.float64
    X = np.ascontiguousarray(X, dtype=ft)
    y = np.ascontiguousarray(y, dtype=ft)
    if X.ndim != 3:
        raise InvalidInputError(f"X must be 3-D (B, n, p), got shape {X.shape}")
    B, n, p = X.shape
    if n < 1 or p < 1:
        raise InvalidInputError(f"need m >= 1 and d >= 1, got {n} x {p}")
    if y.shape != (B, n):
        raise DimensionMismatchError(f"y has shape {y.shape}, expected {(B, n)}")
    lam = np.array(np.broadcast_to(np.asarray(lam, dtype=ft), (B,)), dtype=ft)
    return X, y, lam


def _validate_device(X, y, lam, nlam=None, f32=False):
    import torch

    ft = torch.float32 if f32 else torch.float64
    if X.dtype != ft or y.dtype != ft:
        raise InvalidInputError("device inputs must be float64 (or float32 X and y for the fp32 mode)")
    if X.dim() != 3:
        raise InvalidInputError(f"X must be 3-D (B, n, p), got shape {tuple(X.shape)}")
    B, n, p = X.shape
    if tuple(y.shape) != (B, n):
        raise DimensionMismatchError(f"y has shape {tuple(y.shape)}, expected {(B, n)}")
    nl = B if nlam is None else nlam
    if not torch.is_tensor(lam):
        lam = torch.full((nl,), float(lam), dtype=ft, device=X.device)
    lam = lam.to(device=X.device, dtype=ft).reshape(-1).expand(nl).contiguous()
    return X.contiguous(), y.contiguous(), lam


def _brackets_arg(brackets, B, device=None):
    """(B, 2) float64 per-problem (lo, hi), numpy for the host path or a CUDA tensor for the device path."""
    if brackets is None:
        return None
    if device is not None:
        import torch

        b = torch.as_tensor(brackets, device=device).to(torch.float64).reshape(-1, 2).contiguous()
    else:
        b = np.ascontiguousarray(np.asarray(brackets, dtype=np.float64).reshape(-1, 2))
    if b.shape[0] != B:
        raise DimensionMismatchError(f"brackets has {b.shape[0]} rows for {B} problems")
    return b


def solve_locus_batched(X, y, lam, cfg: LocusConfig | None = None, *, lambda_floor: float = DEFAULT_LAMBDA_FLOOR,
                        data_index=None, brackets=None, strict: bool = False, stream=None,
                        seen_capacity: int = 0) -> BatchedSolveResult:
    """Batched ``solve_locus`` (locus.py:300).  Inputs numpy (host) or CUDA torch tensors.

    float64 inputs run the reference's arithmetic (bit-exact); a float32 X selects
    the fp32 mode (binary32 descents, binary64 outer search; include/ladlasso_b200.h).
    ``brackets`` (B, 2): a per-problem ``LocusConfig.initial_bracket`` (fp64 only).
    Outputs are float64 either way.  Problems whose curve-point scratch overflows
    (status 3, only for searches that stall far past their tolerance) are re-run with
    the worst-case capacity on the host path and whenever ``strict`` is set."""
    res = _solve_locus_once(X, y, lam, cfg, lambda_floor, data_index, brackets, stream, seen_capacity)
    host = not _is_torch(res.status)
    if (host or strict) and seen_capacity == 0:
        st = np.asarray(res.status.cpu() if not host else res.status)
        redo = np.nonzero(st == STATUS_SCRATCH)[0]
        if redo.size:
            res = _rerun_scratch(res, redo, X, y, lam, cfg, lambda_floor, data_index, brackets, stream)
    if strict:
        res.raise_for_status()
    return res


def _rerun_scratch(res, redo, X, y, lam, cfg, lambda_floor, data_index, brackets, stream):
    """Re-solve the status-3 problems with the worst-case curve-point capacity and splice them in."""
    import torch

    on_dev = _is_torch(X)
    idx = torch.as_tensor(redo, device=X.device) if on_dev else redo
    B = res.objective.shape[0]
    lam_all = lam if (on_dev or np.ndim(lam)) else np.full(B, float(lam))
    if data_index is not None:
        di = data_index[idx] if on_dev else np.asarray(data_index)[redo]
        Xs, ys = X, y
    else:
        di = None
        Xs, ys = X[idx], y[idx]
    br = None if brackets is None else (brackets[idx] if on_dev else np.asarray(brackets).reshape(-1, 2)[redo])
    lam_s = lam_all[idx] if on_dev else np.asarray(np.broadcast_to(lam_all, (B,)))[redo]
    p = X.shape[2]
    prm = locus_params(cfg if cfg is not None else LocusConfig(), lambda_floor, p)
    cap = _worst_case_seen(prm)
    sub = _solve_locus_once(Xs, ys, lam_s, cfg, lambda_floor, di, br, stream, cap)
    for f in ("beta", "objective", "iterations", "objective_evals", "converged", "status", "descents", "steps"):
        getattr(res, f)[idx] = getattr(sub, f)
    return res


def _worst_case_seen(prm) -> int:
    outer = 2 * prm.outer_max_iterations if prm.outer_search == 0 else prm.outer_probes * prm.outer_max_iterations
    return max(2 + 3 * 60 + outer + 1, 1 + 12 + 64)


def _solve_locus_once(X, y, lam, cfg, lambda_floor, data_index, brackets, stream, seen_capacity):
    L = _lib.load()
    cfg = cfg if cfg is not None else LocusConfig()
    solver_id = "locus_ternary" if cfg.outer_search == "ternary" else "locus_quadrature"
    f32 = _is_f32(X)
    if brackets is not None and f32:
        raise InvalidInputError("per-problem brackets are implemented for float64 problems")
    if _is_torch(X):
        import torch

        if data_index is not None:  # bounds are checked in the kernel (status 2): no host sync here
            data_index = torch.as_tensor(data_index, device=X.device).to(torch.int64).reshape(-1).contiguous()
        X, y, lam = _validate_device(X, y, lam, None if data_index is None else data_index.shape[0], f32)
        Bd, n, p = X.shape
        B = lam.shape[0]
        prm = locus_params(cfg, lambda_floor, p)
        prm.seen_capacity = int(seen_capacity)
        br = _brackets_arg(brackets, B, X.device)
        dev = X.device
        beta = torch.empty((B, p), dtype=torch.float64, device=dev)
        obj = torch.empty(B, dtype=torch.float64, device=dev)
        it = torch.empty(B, dtype=torch.int32, device=dev)
        ev = torch.empty(B, dtype=torch.int32, device=dev)
        cv = torch.empty(B, dtype=torch.uint8, device=dev)
        stt = torch.empty(B, dtype=torch.uint8, device=dev)
        dsc = torch.empty(B, dtype=torch.int32, device=dev)
        stp = torch.empty(B, dtype=torch.int64, device=dev)
        out = _lib.LocusOut(beta.data_ptr(), obj.data_ptr(), it.data_ptr(), ev.data_ptr(), cv.data_ptr(),
                            stt.data_ptr(), dsc.data_ptr(), stp.data_ptr())
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        t0 = time.perf_counter()
        di = data_index.data_ptr() if data_index is not None else None
        if br is not None:
            _check(L.lad_locus_solve_bracketed_f64(X.data_ptr(), y.data_ptr(), lam.data_ptr(), di, Bd, B, n, p,
                                                   br.data_ptr(), C.byref(prm), C.byref(out), s))
        else:
            fn = L.lad_locus_solve_f32 if f32 else L.lad_locus_solve_f64
            _check(fn(X.data_ptr(), y.data_ptr(), lam.data_ptr(), di, Bd, B, n, p, C.byref(prm), C.byref(out), s))
        return BatchedSolveResult(beta, obj, it, ev, cv.bool(), stt, dsc, stp, solver_id, time.perf_counter() - t0)
    X, y, lam0 = _validate_host(X, y, 0.0, f32)
    Bd, n, p = X.shape
    if data_index is not None:
        data_index = np.ascontiguousarray(data_index, dtype=np.int64)
        if data_index.size and (data_index.min() < 0 or data_index.max() >= Bd):
            raise InvalidInputError("data_index out of range")
        B = data_index.shape[0]
    else:
        B = Bd
    ft = np.float32 if f32 else np.float64
    lam = np.array(np.broadcast_to(np.asarray(lam, dtype=ft), (B,)), dtype=ft)
    prm = locus_params(cfg, lambda_floor, p)
    prm.seen_capacity = int(seen_capacity)
    br = _brackets_arg(brackets, B)
    beta = _host_empty((B, p))
    obj = _host_empty(B)
    it = _host_empty(B, np.int32)
    ev = _host_empty(B, np.int32)
    cv = _host_empty(B, np.uint8)
    stt = _host_empty(B, np.uint8)
    dsc = _host_empty(B, np.int32)
    stp = _host_empty(B, np.int64)
    out = _lib.LocusOut(*(a.ctypes.data for a in (beta, obj, it, ev, cv, stt, dsc, stp)))
    t0 = time.perf_counter()
    di = None if data_index is None else data_index.ctypes.data
    if br is not None:
        _check(L.lad_locus_solve_bracketed_host_f64(X.ctypes.data, y.ctypes.data, lam.ctypes.data, di, Bd, B, n, p,
                                                    br.ctypes.data, C.byref(prm), C.byref(out), stream))
    else:
        fn = L.lad_locus_solve_host_f32 if f32 else L.lad_locus_solve_host_f64
        _check(fn(X.ctypes.data, y.ctypes.data, lam.ctypes.data, di, Bd, B, n, p, C.byref(prm), C.byref(out), stream))
    return BatchedSolveResult(beta, obj, it, ev, cv.astype(bool), stt, dsc, stp, solver_id, time.perf_counter() - t0)


def ccd_descend_batched(X, y, lam, start, cfg: CcdConfig | None = None, frozen=None, *,
                        lambda_floor: float = DEFAULT_LAMBDA_FLOOR) -> BatchedSolveResult:
    """Batched ``ccd_descend`` (ccd.py:126).  ``frozen``: int, None or (B,) array (-1 = none)."""
    import torch

    L = _lib.load()
    cfg = cfg if cfg is not None else CcdConfig()
    if getattr(cfg, "line_search", "exact_median") != "exact_median":
        raise InvalidInputError("the CUDA path implements line_search='exact_median' only")
    host = not _is_torch(X)
    f32 = _is_f32(X)
    if host:
        X, y, lam = _validate_host(X, y, lam, f32)
        dev = torch.device("cuda")
        Xt, yt, lt = (_to_device(a, dev) for a in (X, y, lam))
    else:
        Xt, yt, lt = _validate_device(X, y, lam, None, f32)
        dev = Xt.device
    B, n, p = Xt.shape
    st = torch.as_tensor(np.array(start, dtype=np.float64) if not _is_torch(start) else start,
                         dtype=torch.float64, device=dev).reshape(-1, p).expand(B, p).contiguous()
    if frozen is None and getattr(cfg, "frozen_axis", None) is not None:
        frozen = cfg.frozen_axis
    if frozen is None:
        fr = torch.full((B,), -1, dtype=torch.int32, device=dev)
    else:
        fr = torch.as_tensor(frozen if _is_torch(frozen) else np.asarray(frozen), device=dev).to(torch.int32)
        fr = fr.reshape(-1).expand(B).contiguous()
        frc = fr.cpu().numpy()
        if ((frc < -1) | (frc >= p)).any():
            raise InvalidInputError(f"frozen_axis out of range for d={p}")
    beta = torch.empty((B, p), dtype=torch.float64, device=dev)
    obj = torch.empty(B, dtype=torch.float64, device=dev)
    it = torch.empty(B, dtype=torch.int32, device=dev)
    ev = torch.empty(B, dtype=torch.int32, device=dev)
    cv = torch.empty(B, dtype=torch.uint8, device=dev)
    stt = torch.empty(B, dtype=torch.uint8, device=dev)
    out = _lib.LocusOut(beta.data_ptr(), obj.data_ptr(), it.data_ptr(), ev.data_ptr(), cv.data_ptr(),
                        stt.data_ptr(), None, None)
    s = torch.cuda.current_stream(dev).cuda_stream
    t0 = time.perf_counter()
    fn = L.lad_ccd_descend_f32 if f32 else L.lad_ccd_descend_f64
    _check(fn(Xt.data_ptr(), yt.data_ptr(), lt.data_ptr(), B, n, p, st.data_ptr(), fr.data_ptr(),
              float(cfg.sweep_tolerance), int(cfg.max_sweeps), float(lambda_floor), C.byref(out), s))
    res = BatchedSolveResult(beta, obj, it, ev, cv.bool(), stt, None, None, "ccd_plain", 0.0)
    if host:
        torch.cuda.synchronize(dev)
        res = BatchedSolveResult(_to_host(beta), _to_host(obj), _to_host(it), _to_host(ev),
                                 _to_host(cv.bool()), _to_host(stt), None, None, "ccd_plain",
                                 time.perf_counter() - t0)
    return res


def solve_brute_batched(X, y, lam, max_variables: int = 6, max_candidates: int = 2_000_000, *,
                        lambda_floor: float = DEFAULT_LAMBDA_FLOOR):
    """Batched ``solve_brute`` (brute.py:106).  Returns (beta, objective, vertices)."""
    import torch

    L = _lib.load()
    host = not _is_torch(X)
    if host:
        X, y, lam = _validate_host(X, y, lam)
        dev = torch.device("cuda")
        Xt, yt, lt = (_to_device(a, dev) for a in (X, y, lam))
    else:
        Xt, yt, lt = _validate_device(X, y, lam)
        dev = Xt.device
    B, n, p = Xt.shape
    beta = torch.empty((B, p), dtype=torch.float64, device=dev)
    obj = torch.empty(B, dtype=torch.float64, device=dev)
    nv = torch.empty(B, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    _check(L.lad_brute_solve_f64(Xt.data_ptr(), yt.data_ptr(), lt.data_ptr(), B, n, p, int(max_variables),
                                 int(max_candidates), float(lambda_floor), beta.data_ptr(), obj.data_ptr(),
                                 nv.data_ptr(), s))
    if host:
        return _to_host(beta), _to_host(obj), _to_host(nv)
    return beta, obj, nv


def fp32_peak_tflops() -> float:
    """Measured dense FFMA throughput of the current device (fp32-mode roofline denominator)."""
    import torch

    v = C.c_double()
    _check(_lib.load().lad_fp32_peak_tflops(C.byref(v), torch.cuda.current_stream().cuda_stream))
    return v.value


def fp64_peak_tflops() -> float:
    """Measured dense DFMA throughput of the current device (roofline denominator)."""
    import torch

    v = C.c_double()
    _check(_lib.load().lad_fp64_peak_tflops(C.byref(v), torch.cuda.current_stream().cuda_stream))
    return v.value


def evaluate_objective_batched(X, y, lam, beta, *, lambda_floor: float = DEFAULT_LAMBDA_FLOOR):
    """Batched ``evaluate_objective`` (model.py:151) on the device."""
    import torch

    L = _lib.load()
    host = not _is_torch(X)
    if host:
        X, y, lam = _validate_host(X, y, lam)
        dev = torch.device("cuda")
        Xt, yt, lt = (_to_device(a, dev) for a in (X, y, lam))
        bt = _to_device(np.asarray(beta, dtype=np.float64), dev)
    else:
        Xt, yt, lt = _validate_device(X, y, lam)
        dev = Xt.device
        bt = beta.to(torch.float64).contiguous()
    B, n, p = Xt.shape
    out = torch.empty(B, dtype=torch.float64, device=dev)
    _check(L.lad_objective_f64(Xt.data_ptr(), yt.data_ptr(), lt.data_ptr(), B, n, p, bt.data_ptr(),
                               float(lambda_floor), out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    return _to_host(out) if host else out


def axiswise_minimum_batched(X, y, lam, beta, skip=None, tol: float = 1e-9, *,
                             lambda_floor: float = DEFAULT_LAMBDA_FLOOR):
    """Batched ``is_axiswise_minimum`` (ccd.py:214) on the device: bool per problem.

    ``skip``: None, one axis for all problems, or (B,) axes (-1 = none)."""
    import torch

    L = _lib.load()
    host = not _is_torch(X)
    if host:
        X, y, lam = _validate_host(X, y, lam)
        dev = torch.device("cuda")
        Xt, yt, lt = (_to_device(a, dev) for a in (X, y, lam))
    else:
        Xt, yt, lt = _validate_device(X, y, lam)
        dev = Xt.device
    B, n, p = Xt.shape
    bt = torch.as_tensor(beta if _is_torch(beta) else np.array(beta, dtype=np.float64), dtype=torch.float64,
                         device=dev).reshape(-1, p).expand(B, p).contiguous()
    sk = None
    if skip is not None:
        sk = torch.as_tensor(skip if _is_torch(skip) else np.asarray(skip), device=dev).to(torch.int32)
        sk = sk.reshape(-1).expand(B).contiguous()
    out = torch.empty(B, dtype=torch.uint8, device=dev)
    _check(L.lad_axiswise_minimum_f64(Xt.data_ptr(), yt.data_ptr(), lt.data_ptr(), B, n, p, bt.data_ptr(),
                                      None if sk is None else sk.data_ptr(), float(tol), float(lambda_floor),
                                      out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    if host:
        o = _to_host(out)
        if (o == 2).any():
            raise InvalidInputError(f"problem {int(np.nonzero(o == 2)[0][0])}: non-finite input")
        return o == 1
    return out == 1


# ---------------------------------------------------------------------------
# single-problem mirrors of the reference API (B = 1 calls)
# ---------------------------------------------------------------------------

def _frozen_array(values, ndim, what):
    out = np.array(values, dtype=float)
    if out.ndim != ndim:
        raise InvalidInputError(f"{what} must be {ndim}-D, got shape {out.shape}")
    if not np.isfinite(out).all():
        raise InvalidInputError(f"{what} must contain only finite values")
    out.setflags(write=False)
    return out


@dataclass(frozen=True, eq=False)
class Dataset:
    """model.Dataset (model.py:42-66)."""

    x: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        x = _frozen_array(self.x, 2, "x")
        y = _frozen_array(self.y, 1, "y")
        m, d = x.shape
        if m < 1 or d < 1:
            raise InvalidInputError(f"need m >= 1 and d >= 1, got {m} x {d}")
        if y.shape[0] != m:
            raise DimensionMismatchError(f"y has {y.shape[0]} entries for {m} data rows")
        object.__setattr__(self, "x", x)
        object.__setattr__(self, "y", y)

    @property
    def m(self):
        return self.x.shape[0]

    @property
    def d(self):
        return self.x.shape[1]


@dataclass(frozen=True, eq=False)
class Coefficients:
    beta: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "beta", _frozen_array(self.beta, 1, "beta"))

    def __len__(self):
        return self.beta.shape[0]

    @classmethod
    def zeros(cls, d):
        return cls(np.zeros(d))


@dataclass(frozen=True, eq=False)
class ProblemSpec:
    """model.ProblemSpec (model.py:86-110)."""

    data: Dataset
    lam: float
    lambda_floor: float = DEFAULT_LAMBDA_FLOOR

    def __post_init__(self):
        if not math.isfinite(self.lam) or self.lam < 0:
            raise InvalidInputError("lam must be finite and >= 0")
        if not math.isfinite(self.lambda_floor) or self.lambda_floor <= 0:
            raise InvalidInputError("lambda_floor must be finite and > 0")

    @property
    def lambda_eff(self):
        return max(self.lam, self.lambda_floor)

    @property
    def m(self):
        return self.data.m

    @property
    def d(self):
        return self.data.d


@dataclass(frozen=True, eq=False)
class SolveResult:
    beta: Coefficients
    objective: float
    solver_id: str
    iterations: int
    objective_evals: int
    wall_time: float
    converged: bool


def _spec_arrays(spec):
    data = spec.data
    return (np.asarray(data.x, dtype=float)[None], np.asarray(data.y, dtype=float)[None],
            np.array([float(spec.lam)]), float(getattr(spec, "lambda_floor", DEFAULT_LAMBDA_FLOOR)))


def solve_locus(spec, cfg=None) -> SolveResult:
    """Drop-in for ``ladlasso.locus.solve_locus`` on one problem (runs on the GPU)."""
    X, y, lam, floor = _spec_arrays(spec)
    r = solve_locus_batched(X, y, lam, cfg, lambda_floor=floor, strict=True)
    return SolveResult(Coefficients(r.beta[0]), float(r.objective[0]), r.solver_id, int(r.iterations[0]),
                       int(r.objective_evals[0]), r.wall_time, bool(r.converged[0]))


def ccd_descend(spec, start, cfg=None) -> SolveResult:
    """Drop-in for ``ladlasso.ccd.ccd_descend`` on one problem (runs on the GPU)."""
    X, y, lam, floor = _spec_arrays(spec)
    b = start.beta if hasattr(start, "beta") else np.asarray(start, dtype=float)
    if b.shape != (X.shape[2],):
        raise DimensionMismatchError(f"beta has shape {b.shape}, problem has {X.shape[2]} variables")
    cfg = cfg if cfg is not None else CcdConfig()
    r = ccd_descend_batched(X, y, lam, b[None], cfg, frozen=cfg.frozen_axis, lambda_floor=floor)
    return SolveResult(Coefficients(r.beta[0]), float(r.objective[0]), "ccd_plain", int(r.iterations[0]),
                       int(r.objective_evals[0]), r.wall_time, bool(r.converged[0]))


def solve_ccd(spec, cfg=None, start=None) -> SolveResult:
    return ccd_descend(spec, start if start is not None else np.zeros(spec.d), cfg)


def solve_brute(spec, max_variables: int = 6, max_candidates: int = 2_000_000) -> SolveResult:
    """Drop-in for ``ladlasso.brute.solve_brute`` on one problem (runs on the GPU)."""
    X, y, lam, floor = _spec_arrays(spec)
    t0 = time.perf_counter()
    beta, obj, nv = solve_brute_batched(X, y, lam, max_variables, max_candidates, lambda_floor=floor)
    return SolveResult(Coefficients(beta[0]), float(obj[0]), "brute", int(nv[0]), int(nv[0]),
                       time.perf_counter() - t0, True)


def evaluate_objective(spec, beta) -> float:
    X, y, lam, floor = _spec_arrays(spec)
    b = beta.beta if hasattr(beta, "beta") else np.asarray(beta, dtype=float)
    if b.shape != (X.shape[2],):
        raise DimensionMismatchError(f"beta has shape {b.shape}, problem has {X.shape[2]} variables")
    return float(evaluate_objective_batched(X, y, lam, b[None], lambda_floor=floor)[0])


def is_axiswise_minimum(spec, beta, skip=None, tol: float = 1e-9) -> bool:
    """Drop-in for ``ladlasso.ccd.is_axiswise_minimum`` (runs on the GPU)."""
    X, y, lam, floor = _spec_arrays(spec)
    b = beta.beta if hasattr(beta, "beta") else np.asarray(beta, dtype=float)
    if b.shape != (X.shape[2],):
        raise DimensionMismatchError(f"beta has shape {b.shape}, problem has {X.shape[2]} variables")
    return bool(axiswise_minimum_batched(X, y, lam, b[None], -1 if skip is None else int(skip), tol,
                                         lambda_floor=floor)[0])


def validate_result(spec, result, rtol: float = 1e-12) -> None:
    """Drop-in for ``ladlasso.model.validate_result`` (model.py:180-186): the stored objective must
    reproduce a fresh evaluation (on the GPU) within rtol."""
    f = evaluate_objective(spec, result.beta)
    if abs(result.objective - f) > rtol * max(1.0, abs(f)):
        raise InvalidInputError(f"stored objective {result.objective!r} does not reproduce {f!r}")
