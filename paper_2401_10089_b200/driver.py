"""Public entry point: ``logm(A, opts) -> (L, LogmReport)`` and its batched form.

Mirrors the reference's (missing) driver API -- ``LogmOptions``, ``LogmReport``,
``logm`` (``logmpoly/__init__.py:55``) -- on top of the C ABI
(include/logmpoly_b200.h).  numpy in -> numpy out, torch in -> torch out (same device).
Batches shard by matrix across the given CUDA devices with no collective: each device
runs its contiguous chunk on its own current stream and the shards are gathered.

There is no CPU path: without a CUDA device or without the built library every call
raises (ExtensionMissingError / RuntimeError).
"""
import ctypes
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from . import constants as C
from .exceptions import ConvergenceError, SingularMatrixError, SpectrumError

UNIT_ROUNDOFF = 2.0 ** -53


class OpCounter:
    """Work tally (reference matcore.py:23-48): products (M), divisions (D), thin passes."""

    __slots__ = ("products", "divisions", "estimation_passes")

    def __init__(self, products=0, divisions=0, estimation_passes=0):
        self.products = int(products)
        self.divisions = int(divisions)
        self.estimation_passes = int(estimation_passes)

    @property
    def equivalent_m(self):
        return self.products + 4.0 * self.divisions / 3.0

    def __repr__(self):
        return (f"OpCounter(products={self.products}, divisions={self.divisions}, "
                f"estimation_passes={self.estimation_passes})")


@dataclass
class LogmOptions:
    """SPEC.md:434-437.  ``max_k`` defaults to 5: only schemes k = 1..5 ship with the
    reference."""

    max_k: int = C.K_MAX
    maxiter: int = 40
    balance: bool = True
    theta_table: Optional[Sequence[float]] = None
    db_maxiter: int = 50
    est_itmax: int = 5
    raise_on_error: bool = True
    # eig_small pre-check: off by default (caller contract);
    # when on, matrices with n <= spectrum_cap and an eigenvalue on the closed negative real
    # axis get status SPECTRUM (-> SpectrumError)
    check_spectrum: bool = False
    spectrum_cap: int = 512

    def theta(self):
        return tuple(self.theta_table) if self.theta_table is not None else C.THETA


@dataclass
class LogmReport:
    """SPEC.md:438-443 plus the GPU report's status / margin fields."""

    s: int = 0
    k_selected: int = 0
    alpha_used: float = 0.0
    counter: OpCounter = field(default_factory=OpCounter)
    norm_estimations: int = 0
    balanced: bool = True
    status: int = 0
    db_iters: int = 0
    balance_sweeps: int = 0
    min_margin: float = float("inf")
    db_plateau: int = 0

    @classmethod
    def from_record(cls, r):
        return cls(s=int(r["s"]), k_selected=int(r["k"]), alpha_used=float(r["alpha_used"]),
                   counter=OpCounter(r["products"], r["divisions"], r["estimation_passes"]),
                   norm_estimations=int(r["norm_estimations"]), balanced=bool(r["balanced"]),
                   status=int(r["status"]), db_iters=int(r["db_iters"]),
                   balance_sweeps=int(r["balance_sweeps"]), min_margin=float(r["min_margin"]),
                   db_plateau=int(r["db_plateau"]))


def _torch():
    import torch
    return torch


def _c_opts(opts):
    o = _lib.Opts()
    _lib.load().lgm_default_opts(ctypes.byref(o))
    o.max_k = int(opts.max_k)
    o.maxiter_s = int(opts.maxiter)
    o.db_maxiter = int(opts.db_maxiter)
    o.est_itmax = int(opts.est_itmax)
    o.balance = 1 if opts.balance else 0
    th = (ctypes.c_double * C.K_MAX)(*[float(t) for t in opts.theta()][:C.K_MAX])
    o.theta = ctypes.cast(th, ctypes.POINTER(ctypes.c_double))
    return o, th


def _as_batch(A):
    """Validate like as_square (matcore.py:51-66); returns (tensor-like, was_numpy, squeeze)."""
    torch = _torch()
    if isinstance(A, torch.Tensor):
        if A.dim() not in (2, 3) or A.shape[-1] != A.shape[-2] or A.shape[-1] < 1:
            raise ValueError(f"matrix must be square, got shape {tuple(A.shape)}")
        if A.is_complex():
            raise ValueError("complex input is not supported by the FP64 GPU path")
        squeeze = A.dim() == 2
        return (A.unsqueeze(0) if squeeze else A), False, squeeze
    A = np.asarray(A)
    if A.ndim not in (2, 3) or A.shape[-1] != A.shape[-2] or A.shape[-1] < 1:
        raise ValueError(f"matrix must be square, got shape {A.shape}")
    if np.iscomplexobj(A):
        raise ValueError("complex input is not supported by the FP64 GPU path")
    squeeze = A.ndim == 2
    A = np.ascontiguousarray(A, dtype=np.float64)
    return (A[None] if squeeze else A), True, squeeze


def _raise_for(rep, idx):
    st = int(rep["status"])
    msg = _lib.status_string(st)
    where = f" (matrix {idx})" if idx is not None else ""
    report = LogmReport.from_record(rep)
    if st == _lib.SINGULAR:
        raise SingularMatrixError(msg + where)
    if st in (_lib.DB_NOCONV, _lib.SCALING_MAXITER):
        raise ConvergenceError(msg + where, report)
    if st == _lib.NONFINITE:
        raise ValueError(msg + where)
    if st == _lib.SPECTRUM:
        raise SpectrumError(msg + where)
    raise RuntimeError(msg + where)


def run_device(A_dev, opts, stream=None):
    """Run lgm_logm_f64 on one device tensor (B, n, n) float64 contiguous.
    Returns (L_dev, report_dev uint8 tensor (B*56,)).  Stream-ordered, no sync."""
    torch = _torch()
    lib = _lib.load()
    B, n, _ = A_dev.shape
    dev = A_dev.device
    L = torch.empty_like(A_dev)
    rep = torch.empty(max(B, 1) * _lib.REPORT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    ws_bytes = ctypes.c_size_t(0)
    _lib.check(lib.lgm_workspace_bytes(n, B, ctypes.byref(ws_bytes)), "lgm_workspace_bytes")
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    ws = _workspace(dev, stream, n, B, int(ws_bytes.value))
    o, keep = _c_opts(opts)
    rc = lib.lgm_logm_f64(A_dev.data_ptr(), L.data_ptr(), n, B, n, ctypes.byref(o), rep.data_ptr(),
                          ws.data_ptr(), ws_bytes.value, ctypes.c_void_p(stream.cuda_stream))
    del keep
    _lib.check(rc, "lgm_logm_f64")
    return L, rep, ws


# per-thread caches (streams, pinned report staging): concurrent callers on different threads
# never share them, so logm_batched stays reentrant like the reference's pure functions
_TLS = threading.local()


def _workspace(dev, stream, n, B, nbytes):
    """Per-(thread, device, stream, shape) workspace, reused across calls: Engine G caches
    its CUDA graph per workspace address, so a stable workspace means one capture per shape
    (calls on one stream are ordered, so reuse is safe).  Small LRU per thread."""
    cache = getattr(_TLS, "ws", None)
    if cache is None:
        cache = _TLS.ws = {}
    key = (dev.index, int(stream.cuda_stream), n, B)
    ws = cache.pop(key, None)
    if ws is None:
        with _torch().cuda.stream(stream):  # owned by `stream`: eviction reuse stays stream-ordered
            ws = _torch().empty(max(nbytes, 1), dtype=_torch().uint8, device=dev)
        while len(cache) >= 6:
            cache.pop(next(iter(cache)))
    cache[key] = ws
    return ws


def _host_chunks(B, n):
    """Chunking of a host-resident batch for the copy/compute pipeline: Engine F launches
    (n <= lgm_max_fused_n) of >= ~680 matrices on their own streams (the chunk kernels
    overlap each other on the device) so the H2D of chunk i+1 and the D2H of chunk i-1
    overlap chunk i's kernel (config 2, 2.56 ms kernel: 1 chunk 3.91 ms, 3: 3.11, 4: 3.07,
    6: 2.98, 8: 3.07).  Engine G keeps one chunk: its batch parallelism is what fills the GPU
    (a chunk of the config-4 batch would run its inversions on fewer SMs)."""
    if n > int(_lib.load().lgm_max_fused_n()):
        return 1
    return max(1, min(6, B // 680))


def _streams(dev, count):
    cache = getattr(_TLS, "streams", None)
    if cache is None:
        cache = _TLS.streams = {}
    key = (dev.index, count)
    if key not in cache:
        cache[key] = [_torch().cuda.Stream(dev) for _ in range(count)]
    return cache[key]


def _rep_staging(nbytes):
    """Pinned staging for the per-matrix reports (per thread, reused: a pinned allocation
    costs ~1 ms)."""
    buf = getattr(_TLS, "rep", None)
    if buf is None or buf.numel() < nbytes:
        buf = _torch().empty(max(nbytes, 1 << 16), dtype=_torch().uint8, pin_memory=True)
        _TLS.rep = buf
    return buf


def logm_batched(A, opts=None, devices=None, out=None):
    """Batched principal logarithm of (B, n, n) (or (n, n)) float64 matrices.

    Returns (L, reports) where ``reports`` is a numpy structured array (REPORT_DTYPE), one
    record per matrix.  With ``opts.raise_on_error`` (default) the first failing matrix
    raises the reference's exception type.  ``out``: optional host buffer for L when the
    input is on the host (numpy array or CPU tensor of the input's shape, float64,
    contiguous; pinned memory lets the copies overlap the kernels) -- repeated callers
    pass one to avoid a pinned allocation per call.
    """
    torch = _torch()
    opts = opts or LogmOptions()
    Ab, was_numpy, squeeze = _as_batch(A)
    if not torch.cuda.is_available():
        raise RuntimeError("logm needs a CUDA device (B200); there is no CPU fallback")
    if devices is None:
        if not was_numpy and Ab.is_cuda:
            devices = [Ab.device]
        else:
            devices = [torch.device("cuda", torch.cuda.current_device())]
    devices = [torch.device(d) for d in devices]
    B = Ab.shape[0]
    G = len(devices)
    n = Ab.shape[-1]
    bounds = [(g * B) // G for g in range(G + 1)]
    isz = _lib.REPORT_DTYPE.itemsize
    # reports always go to (pinned) host memory; L to pinned host memory for numpy / CPU
    # tensor input (chunked H2D -> kernel -> D2H pipeline, one stream per chunk), else it
    # stays on the device (no copy when a single shard already lives there)
    rep_host = _rep_staging(max(B, 1) * isz)
    to_host = was_numpy or not Ab.is_cuda
    if to_host:
        if out is None:
            Lh = torch.empty((B, n, n), dtype=torch.float64, pin_memory=True)
        else:
            Lh = torch.from_numpy(out) if isinstance(out, np.ndarray) else out
            if (tuple(Lh.shape[-3:] if Lh.dim() == 3 else (1,) + tuple(Lh.shape)) != (B, n, n)
                    or Lh.dtype != torch.float64 or Lh.is_cuda or not Lh.is_contiguous()):
                raise ValueError("out must be a contiguous float64 host buffer of the input's shape")
            Lh = Lh.view(B, n, n)
        host = (torch.from_numpy(Ab) if was_numpy else Ab.to(torch.float64)).contiguous()
    outs = []
    for g, dev in enumerate(devices):
        lo, hi = bounds[g], bounds[g + 1]
        if hi == lo:
            continue
        with torch.cuda.device(dev):
            if to_host:
                nc = _host_chunks(hi - lo, n)
                cb = [lo + ((hi - lo) * c) // nc for c in range(nc + 1)]
                cur = torch.cuda.current_stream(dev)
                for c, s in enumerate(_streams(dev, nc)):
                    a, b = cb[c], cb[c + 1]
                    s.wait_stream(cur)
                    with torch.cuda.stream(s):
                        Ad = host[a:b].to(dev, non_blocking=True)
                        L, rep, ws = run_device(Ad, opts, s)
                        Lh[a:b].copy_(L, non_blocking=True)
                        rep_host[a * isz:b * isz].copy_(rep[:(b - a) * isz], non_blocking=True)
                    outs.append((a, b, dev, L, rep, Ad, ws))
            else:
                Ad = Ab[lo:hi].to(device=dev, dtype=torch.float64).contiguous()
                L, rep, ws = run_device(Ad, opts)
                rep_host[lo * isz:hi * isz].copy_(rep[:(hi - lo) * isz], non_blocking=True)
                outs.append((lo, hi, dev, L, rep, Ad, ws))
    for dev in {o[2] for o in outs}:
        torch.cuda.synchronize(dev)
    reports = rep_host[:B * isz].numpy().copy().view(_lib.REPORT_DTYPE)
    if opts.check_spectrum and B and n <= opts.spectrum_cap:
        from .validate import spectrum_violations
        bad = spectrum_violations(Ab if not was_numpy else torch.from_numpy(Ab), opts.spectrum_cap)
        reports["status"][bad] = _lib.SPECTRUM
    if to_host:
        if out is not None:
            Lout = out.reshape(B, n, n) if isinstance(out, np.ndarray) else Lh
        else:
            Lout = Lh.numpy() if was_numpy else Lh
    elif len(outs) == 1 and outs[0][2] == Ab.device:
        Lout = outs[0][3]
    else:
        Lout = torch.cat([o[3].to(Ab.device) for o in outs]) if outs else torch.empty_like(Ab)
    if opts.raise_on_error:
        bad = np.nonzero(reports["status"] != 0)[0]
        if bad.size:
            _raise_for(reports[bad[0]], None if squeeze else int(bad[0]))
    if squeeze:
        Lout = Lout[0]
    return Lout, reports


def logm(A, opts=None):
    """Principal matrix logarithm of one square float64 matrix.

    Returns (L, LogmReport).  Raises SingularMatrixError, ConvergenceError (with the
    partial report) or ValueError like the reference.
    """
    L, reps = logm_batched(A, opts)
    if getattr(L, "ndim", None) == 3 or (hasattr(L, "dim") and L.dim() == 3):
        if L.shape[0] != 1:
            raise ValueError("logm takes one matrix; use logm_batched for (B, n, n)")
        L = L[0]
    return L, LogmReport.from_record(reps[0])


def unbalance_postprocess(L, scale):
    """L <- T L T^-1 (matcore.py:175-177).  Exact for radix-2 scales."""
    scale = np.asarray(scale, dtype=np.float64)
    return L * (scale[:, None] / scale[None, :])
