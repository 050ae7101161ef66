"""Thin ctypes binding of libnef (include/nef.h).  Argument marshalling only: every step
of the MU sweep runs in the library's sm_100a kernels.  PyTorch supplies device memory and
streams.  There is NO CPU fallback: if libnef.so is missing this module raises on import.

Functions carry the C ABI's names (``nef_plan``, ``nef_fit``, ``nef_loss`` ...); ``Plan`` is
a small convenience wrapper over them.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NEF_LIB") or os.path.join(_HERE, "libnef.so")   # NEF_LIB: diagnostic builds

NEF_STATUS = {0: "OK", 1: "PARSE", 2: "SHAPE", 3: "DOMAIN", 4: "DATA", 5: "ARG", 6: "CUDA", 7: "NCCL",
              8: "UNSUPPORTED"}


class NefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("nef error %s (%d): %s" % (NEF_STATUS.get(code, "?"), code, msg))
        self.code = code
        self.status = NEF_STATUS.get(code, "?")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libnef.so not built (%s); run `make` or __graft_entry__.build()" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    i64p = ctypes.POINTER(ctypes.c_int64)
    vp = ctypes.c_void_p
    d = ctypes.c_double
    sig = {
        "nef_plan": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, i64p, ctypes.c_int, i64p, ctypes.POINTER(vp)]),
        "nef_plan_info": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), i64p, i64p,
                                         ctypes.POINTER(ctypes.c_size_t)]),
        "nef_factor_shape": (ctypes.c_int, [vp, ctypes.c_int, i64p, ctypes.POINTER(ctypes.c_int)]),
        "nef_local_shape": (ctypes.c_int, [vp, i64p, ctypes.POINTER(ctypes.c_int)]),
        "nef_plan_describe": (ctypes.c_int, [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
        "nef_fit": (ctypes.c_int, [vp, vp, vp, d, d, d, vp, ctypes.c_int, ctypes.POINTER(d), vp, ctypes.c_size_t, vp]),
        "nef_update": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, d, d, d, vp, vp, ctypes.c_size_t, vp]),
        "nef_num_den": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, d, d, vp, vp, vp, vp, ctypes.c_size_t, vp]),
        "nef_apply_update": (ctypes.c_int, [vp, ctypes.c_int, d, d, d, vp, vp, vp, vp]),
        "nef_loss": (ctypes.c_int, [vp, vp, vp, d, d, vp, ctypes.POINTER(d), i64p, vp, ctypes.c_size_t, vp]),
        "nef_host_scratch_bytes": (ctypes.c_size_t, [vp, ctypes.c_int]),
        "nef_fit_host": (ctypes.c_int, [vp, vp, vp, d, d, d, vp, ctypes.c_int, ctypes.POINTER(d), vp, ctypes.c_size_t,
                                        vp]),
        "nef_nccl_unique_id": (ctypes.c_int, [vp]),
        "nef_plan_shard": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp]),
        "nef_plan_shard_host": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int]),
        "nef_last_launch_count": (ctypes.c_int64, []),
        "nef_set_kernel_policy": (ctypes.c_int, [ctypes.c_int]),
        "nef_profile_enable": (ctypes.c_int, [ctypes.c_int]),
        "nef_debug_dump": (ctypes.c_int, [vp]),
        "nef_debug_trace": (ctypes.c_int, [vp]),
        "nef_profile_read": (ctypes.c_int, [ctypes.POINTER(d), i64p, ctypes.POINTER(d)]),
        "nef_fit_ex": (ctypes.c_int, [vp, vp, vp, vp, d, vp, ctypes.c_int, ctypes.POINTER(d), vp, ctypes.c_size_t, vp]),
        "nef_fit_split": (ctypes.c_int, [vp, vp, vp, vp, d, vp, vp, ctypes.POINTER(d), i64p, ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_int), vp, ctypes.c_size_t, vp]),
        "nef_update_ex": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, vp, d, vp, vp, ctypes.c_size_t, vp]),
        "nef_num_den_ex": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
        "nef_apply_update_ex": (ctypes.c_int, [vp, ctypes.c_int, vp, d, vp, vp, vp, vp]),
        "nef_loss_ex": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.POINTER(d), i64p, vp, ctypes.c_size_t, vp]),
        "nef_restarts_workspace_bytes": (ctypes.c_size_t, [vp, ctypes.c_int]),
        "nef_fit_restarts": (ctypes.c_int, [vp, vp, vp, vp, d, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(d), vp,
                                            ctypes.c_size_t, vp]),
        "nef_plan_destroy": (None, [vp]),
        "nef_last_error": (ctypes.c_char_p, []),
        "nef_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
EXPORTED = ("nef_plan", "nef_plan_info", "nef_factor_shape", "nef_local_shape", "nef_plan_describe", "nef_fit",
            "nef_update", "nef_num_den", "nef_apply_update", "nef_loss", "nef_host_scratch_bytes", "nef_fit_host",
            "nef_nccl_unique_id", "nef_plan_shard", "nef_plan_shard_host", "nef_last_launch_count",
            "nef_set_kernel_policy",
            "nef_profile_enable", "nef_profile_read", "nef_debug_dump", "nef_debug_trace",
            "nef_fit_ex", "nef_fit_split", "nef_restarts_workspace_bytes", "nef_fit_restarts", "nef_update_ex", "nef_num_den_ex", "nef_apply_update_ex", "nef_loss_ex",
            "nef_plan_destroy", "nef_last_error", "nef_version")

LOSS_KINDS = {"ab": 0, "negbin": 1, "bernoulli": 2, "binomial": 3, "js": 4}
STOP_REASONS = {1: "patience", 2: "plateau", 3: "max_iters"}


class nef_loss_spec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("param", ctypes.c_double), ("aux", ctypes.c_void_p)]


class nef_stop_rule(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int), ("min_rel_decrease", ctypes.c_double), ("val_patience", ctypes.c_int)]


def loss_spec(kind="ab", alpha=1.0, beta=0.0, param=0.0, aux=None):
    """Build an nef_loss_spec: kind in ab / negbin / bernoulli / binomial / js; param = phi (negbin)
    or n (binomial); aux = optional per-entry phi / n CUDA tensor (float32, Y's shape)."""
    return nef_loss_spec(LOSS_KINDS[kind], float(alpha), float(beta), float(param),
                         ctypes.c_void_p(int(aux.data_ptr())) if aux is not None else None)


def _check(code):
    if code != 0:
        raise NefError(code, LIB.nef_last_error().decode())


def _i64(seq):
    seq = [int(x) for x in seq]
    return (ctypes.c_int64 * max(1, len(seq)))(*seq)


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(int(t.data_ptr()))


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    import torch
    return ctypes.c_void_p(int(torch.cuda.current_stream().cuda_stream))


def _validate(h, Y=None, mask=None, factors=None, host=False):
    """Check what the C ABI cannot: dtype, contiguity, device and shape of every tensor (the
    library sees raw pointers only).  Raises NefError(ARG)."""
    import torch

    def bad(msg):
        raise NefError(5, msg)

    def where(t, name):
        if host:
            if t.is_cuda:
                bad("%s must be a host tensor" % name)
        elif not t.is_cuda:
            bad("%s must be a CUDA tensor" % name)
        if not t.is_contiguous():
            bad("%s must be contiguous" % name)

    if Y is not None:
        where(Y, "Y")
        if Y.dtype != torch.float32:
            bad("Y must be float32, got %s" % Y.dtype)
        if tuple(Y.shape) != nef_local_shape(h):
            bad("Y shape %s != plan's local shape %s" % (tuple(Y.shape), nef_local_shape(h)))
    if mask is not None:
        where(mask, "mask")
        if mask.dtype not in (torch.uint8, torch.bool):
            bad("mask must be uint8 or bool, got %s" % mask.dtype)
        if Y is not None and tuple(mask.shape) != tuple(Y.shape):
            bad("mask shape %s != Y shape %s" % (tuple(mask.shape), tuple(Y.shape)))
    if factors is not None:
        n = nef_plan_info(h)["n_factors"]
        if len(factors) != n:
            bad("expected %d factors, got %d" % (n, len(factors)))
        for l, f in enumerate(factors):
            where(f, "factor %d" % l)
            if f.dtype != torch.float32:
                bad("factor %d must be float32, got %s" % (l, f.dtype))
            if tuple(f.shape) != nef_factor_shape(h, l):
                bad("factor %d shape %s != %s" % (l, tuple(f.shape), nef_factor_shape(h, l)))
            if Y is not None and not host and f.device != Y.device:
                bad("factor %d on %s, Y on %s" % (l, f.device, Y.device))


def _validate_nd(h, ell, num, den):
    import torch
    shp = nef_factor_shape(h, ell)
    for name, t in (("num", num), ("den", den)):
        if not t.is_cuda or not t.is_contiguous() or t.dtype != torch.float32 or tuple(t.shape) != shp:
            raise NefError(5, "%s must be a contiguous float32 CUDA tensor of shape %s" % (name, shp))


def _fptrs(factors):
    arr = (ctypes.c_void_p * len(factors))(*[int(f.data_ptr()) for f in factors])
    return arr


# ----------------------------------------------------------------------------- C names
def nef_plan(model: str, shape, ranks):
    h = ctypes.c_void_p()
    _check(LIB.nef_plan(model.encode(), len(shape), _i64(shape), len(ranks), _i64(ranks), ctypes.byref(h)))
    return h


def nef_plan_destroy(h):
    LIB.nef_plan_destroy(h)


def nef_plan_info(h):
    L = ctypes.c_int()
    sm = ctypes.c_int()
    lb = ctypes.c_int64()
    ll = ctypes.c_int64()
    ws = ctypes.c_size_t()
    _check(LIB.nef_plan_info(h, ctypes.byref(L), ctypes.byref(sm), ctypes.byref(lb), ctypes.byref(ll), ctypes.byref(ws)))
    return dict(n_factors=L.value, shard_mode=sm.value, local_begin=lb.value, local_len=ll.value,
                workspace_bytes=ws.value)


def nef_factor_shape(h, ell):
    dims = (ctypes.c_int64 * 8)()
    nd = ctypes.c_int()
    _check(LIB.nef_factor_shape(h, ell, dims, ctypes.byref(nd)))
    return tuple(dims[i] for i in range(nd.value))


def nef_local_shape(h):
    dims = (ctypes.c_int64 * 8)()
    nd = ctypes.c_int()
    _check(LIB.nef_local_shape(h, dims, ctypes.byref(nd)))
    return tuple(dims[i] for i in range(nd.value))


def nef_plan_describe(h):
    n = ctypes.c_size_t()
    _check(LIB.nef_plan_describe(h, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _check(LIB.nef_plan_describe(h, buf, n.value, ctypes.byref(n)))
    return json.loads(buf.value.decode())


def nef_fit(h, Y, mask, alpha, beta, eps, factors, iters, workspace, stream=None, want_trace=True):
    _validate(h, Y, mask, factors)
    trace = (ctypes.c_double * (iters + 1))() if want_trace else None
    _check(LIB.nef_fit(h, _ptr(Y), _ptr(mask), float(alpha), float(beta), float(eps), _fptrs(factors), int(iters),
                       trace, _ptr(workspace), workspace.numel(), _stream(stream)))
    return np.array(trace[:], dtype=np.float64) if want_trace else None


def nef_update(h, ell, Y, mask, alpha, beta, eps, factors, workspace, stream=None):
    _validate(h, Y, mask, factors)
    _check(LIB.nef_update(h, int(ell), _ptr(Y), _ptr(mask), float(alpha), float(beta), float(eps), _fptrs(factors),
                          _ptr(workspace), workspace.numel(), _stream(stream)))


def nef_num_den(h, ell, Y, mask, alpha, beta, factors, num, den, workspace, stream=None):
    _validate(h, Y, mask, factors)
    _validate_nd(h, ell, num, den)
    _check(LIB.nef_num_den(h, int(ell), _ptr(Y), _ptr(mask), float(alpha), float(beta), _fptrs(factors), _ptr(num),
                           _ptr(den), _ptr(workspace), workspace.numel(), _stream(stream)))


def nef_apply_update(h, ell, alpha, beta, eps, factors, num, den, stream=None):
    _validate(h, factors=factors)
    _validate_nd(h, ell, num, den)
    _check(LIB.nef_apply_update(h, int(ell), float(alpha), float(beta), float(eps), _fptrs(factors), _ptr(num),
                                _ptr(den), _stream(stream)))


def nef_loss(h, Y, mask, alpha, beta, factors, workspace, stream=None):
    _validate(h, Y, mask, factors)
    s = ctypes.c_double()
    n = ctypes.c_int64()
    _check(LIB.nef_loss(h, _ptr(Y), _ptr(mask), float(alpha), float(beta), _fptrs(factors), ctypes.byref(s),
                        ctypes.byref(n), _ptr(workspace), workspace.numel(), _stream(stream)))
    return s.value, n.value


def nef_host_scratch_bytes(h, has_mask):
    return int(LIB.nef_host_scratch_bytes(h, 1 if has_mask else 0))


def nef_fit_host(h, Y_host, mask_host, alpha, beta, eps, factors_host, iters, scratch, stream=None):
    """Y_host / mask_host / factors_host: host tensors (ideally pinned), contiguous."""
    _validate(h, Y_host, mask_host, factors_host, host=True)
    trace = (ctypes.c_double * (iters + 1))()
    fp = (ctypes.c_void_p * len(factors_host))(*[int(f.data_ptr()) for f in factors_host])
    _check(LIB.nef_fit_host(h, _ptr(Y_host), _ptr(mask_host), float(alpha), float(beta), float(eps), fp, int(iters),
                            trace, _ptr(scratch), scratch.numel(), _stream(stream)))
    return np.array(trace[:], dtype=np.float64)


def _check_aux(h, spec, aux):
    if aux is not None:
        import torch
        if not aux.is_cuda or not aux.is_contiguous() or aux.dtype != torch.float32 or tuple(aux.shape) != nef_local_shape(h):
            raise NefError(5, "aux must be a contiguous float32 CUDA tensor of Y's local shape")


def nef_fit_ex(h, Y, mask, spec, eps, factors, iters, workspace, stream=None, aux=None):
    _validate(h, Y, mask, factors)
    _check_aux(h, spec, aux)
    trace = (ctypes.c_double * (iters + 1))()
    _check(LIB.nef_fit_ex(h, _ptr(Y), _ptr(mask), ctypes.byref(spec), float(eps), _fptrs(factors), int(iters), trace,
                          _ptr(workspace), workspace.numel(), _stream(stream)))
    return np.array(trace[:], dtype=np.float64)


def nef_fit_split(h, Y, labels, spec, eps, factors, max_iters, min_rel_decrease, val_patience, workspace, stream=None,
                  aux=None):
    """Returns dict(traces=[train, validation, heldout] arrays of sweeps + 1 loss sums, counts, sweeps, reason)."""
    _validate(h, Y, labels, factors)
    _check_aux(h, spec, aux)
    rule = nef_stop_rule(int(max_iters), float(min_rel_decrease), int(val_patience))
    tr = (ctypes.c_double * (3 * (max_iters + 1)))()
    counts = (ctypes.c_int64 * 3)()
    sweeps = ctypes.c_int()
    reason = ctypes.c_int()
    _check(LIB.nef_fit_split(h, _ptr(Y), _ptr(labels), ctypes.byref(spec), float(eps), _fptrs(factors),
                             ctypes.byref(rule), tr, counts, ctypes.byref(sweeps), ctypes.byref(reason),
                             _ptr(workspace), workspace.numel(), _stream(stream)))
    n = sweeps.value
    T = max_iters + 1
    traces = [np.array(tr[q * T:q * T + n + 1], dtype=np.float64) for q in range(3)]
    return dict(traces=traces, counts=[int(c) for c in counts], sweeps=n, reason=STOP_REASONS.get(reason.value, "?"))


def nef_restarts_workspace_bytes(h, restarts):
    return int(LIB.nef_restarts_workspace_bytes(h, int(restarts)))


def nef_fit_restarts(h, Y, mask, spec, eps, restart_factors, iters, workspace, stream=None):
    """restart_factors: list (restarts) of factor lists; returns the loss traces, restarts x (iters + 1)."""
    S = len(restart_factors)
    for F in restart_factors:
        _validate(h, Y, mask, F)
    flat = [f for F in restart_factors for f in F]
    tr = (ctypes.c_double * (S * (iters + 1)))()
    _check(LIB.nef_fit_restarts(h, _ptr(Y), _ptr(mask), ctypes.byref(spec), float(eps), _fptrs(flat), S, int(iters), tr,
                                _ptr(workspace), workspace.numel(), _stream(stream)))
    return np.array(tr[:], dtype=np.float64).reshape(S, iters + 1)


def nef_update_ex(h, ell, Y, mask, spec, eps, factors, workspace, stream=None):
    _validate(h, Y, mask, factors)
    _check(LIB.nef_update_ex(h, int(ell), _ptr(Y), _ptr(mask), ctypes.byref(spec), float(eps), _fptrs(factors),
                             _ptr(workspace), workspace.numel(), _stream(stream)))


def nef_num_den_ex(h, ell, Y, mask, spec, factors, num, den, workspace, stream=None):
    _validate(h, Y, mask, factors)
    _validate_nd(h, ell, num, den)
    _check(LIB.nef_num_den_ex(h, int(ell), _ptr(Y), _ptr(mask), ctypes.byref(spec), _fptrs(factors), _ptr(num),
                              _ptr(den), _ptr(workspace), workspace.numel(), _stream(stream)))


def nef_apply_update_ex(h, ell, spec, eps, factors, num, den, stream=None):
    _validate(h, factors=factors)
    _validate_nd(h, ell, num, den)
    _check(LIB.nef_apply_update_ex(h, int(ell), ctypes.byref(spec), float(eps), _fptrs(factors), _ptr(num), _ptr(den),
                                   _stream(stream)))


def nef_loss_ex(h, Y, mask, spec, factors, workspace, stream=None):
    _validate(h, Y, mask, factors)
    s = ctypes.c_double()
    n = ctypes.c_int64()
    _check(LIB.nef_loss_ex(h, _ptr(Y), _ptr(mask), ctypes.byref(spec), _fptrs(factors), ctypes.byref(s),
                           ctypes.byref(n), _ptr(workspace), workspace.numel(), _stream(stream)))
    return s.value, n.value


def nef_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(LIB.nef_nccl_unique_id(buf))
    return buf.raw


def nef_plan_shard(h, rank, world, uid: bytes | None):
    ub = ctypes.create_string_buffer(uid, 128) if uid is not None else None
    _check(LIB.nef_plan_shard(h, int(rank), int(world), ub))


def nef_plan_shard_host(h, rank, world):
    _check(LIB.nef_plan_shard_host(h, int(rank), int(world)))


def nef_last_launch_count() -> int:
    return int(LIB.nef_last_launch_count())


def nef_set_kernel_policy(policy: int):
    _check(LIB.nef_set_kernel_policy(int(policy)))


def nef_profile_enable(on: bool = True):
    _check(LIB.nef_profile_enable(1 if on else 0))


def nef_profile_read():
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    b = ctypes.c_double()
    _check(LIB.nef_profile_read(ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b)))
    return ms.value, n.value, b.value


def nef_debug_dump(buf):
    _check(LIB.nef_debug_dump(_ptr(buf)))


def nef_debug_trace(buf):
    _check(LIB.nef_debug_trace(_ptr(buf)))


def nef_version() -> str:
    return LIB.nef_version().decode()


# ----------------------------------------------------------------------------- wrapper
class Plan:
    """Owning wrapper: ``Plan(model, shape, ranks)``; workspace allocated lazily with torch."""

    def __init__(self, model, shape, ranks):
        self.model = model
        self.gshape = tuple(int(x) for x in shape)
        self.ranks = tuple(int(x) for x in ranks)
        self.h = nef_plan(model, self.gshape, self.ranks)
        self._ws = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                nef_plan_destroy(h)
            except TypeError:   # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    @property
    def info(self):
        return nef_plan_info(self.h)

    @property
    def n_factors(self):
        return self.info["n_factors"]

    def factor_shape(self, ell):
        return nef_factor_shape(self.h, ell)

    def factor_shapes(self):
        return [self.factor_shape(l) for l in range(self.n_factors)]

    @property
    def local_shape(self):
        return nef_local_shape(self.h)

    def describe(self):
        return nef_plan_describe(self.h)

    def shard(self, rank, world, uid=None):
        nef_plan_shard(self.h, rank, world, uid)
        self._ws = None

    def shard_host(self, rank, world):
        """Host-side split only (no communicator): nef_num_den then returns local partials."""
        nef_plan_shard_host(self.h, rank, world)
        self._ws = None

    def workspace(self, device=None):
        import torch
        need = self.info["workspace_bytes"]
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device or "cuda")
        return self._ws

    def fit(self, Y, mask, alpha, beta, factors, iters, eps=1e-12, stream=None):
        return nef_fit(self.h, Y, mask, alpha, beta, eps, factors, iters, self.workspace(Y.device), stream)

    def update(self, ell, Y, mask, alpha, beta, factors, eps=1e-12, stream=None):
        nef_update(self.h, ell, Y, mask, alpha, beta, eps, factors, self.workspace(Y.device), stream)

    def num_den(self, ell, Y, mask, alpha, beta, factors, stream=None):
        import torch
        shp = self.factor_shape(ell)
        num = torch.empty(shp, dtype=torch.float32, device=Y.device)
        den = torch.empty(shp, dtype=torch.float32, device=Y.device)
        nef_num_den(self.h, ell, Y, mask, alpha, beta, factors, num, den, self.workspace(Y.device), stream)
        return num, den

    def apply_update(self, ell, alpha, beta, factors, num, den, eps=1e-12, stream=None):
        nef_apply_update(self.h, ell, alpha, beta, eps, factors, num, den, stream)

    def loss(self, Y, mask, alpha, beta, factors, stream=None):
        return nef_loss(self.h, Y, mask, alpha, beta, factors, self.workspace(Y.device), stream)

    # any loss of nef_loss_spec: spec = loss_spec("negbin", param=2.0) etc.
    def fit_ex(self, Y, mask, spec, factors, iters, eps=1e-12, stream=None, aux=None):
        return nef_fit_ex(self.h, Y, mask, spec, eps, factors, iters, self.workspace(Y.device), stream, aux)

    def fit_split(self, Y, labels, spec, factors, max_iters=5000, min_rel_decrease=1e-6, val_patience=5, eps=1e-12,
                  stream=None, aux=None):
        return nef_fit_split(self.h, Y, labels, spec, eps, factors, max_iters, min_rel_decrease, val_patience,
                             self.workspace(Y.device), stream, aux)

    def fit_restarts(self, Y, mask, spec, restart_factors, iters, eps=1e-12, stream=None):
        import torch
        need = nef_restarts_workspace_bytes(self.h, len(restart_factors))
        ws = torch.empty(need, dtype=torch.uint8, device=Y.device)
        return nef_fit_restarts(self.h, Y, mask, spec, eps, restart_factors, iters, ws, stream)

    def num_den_ex(self, ell, Y, mask, spec, factors, stream=None):
        import torch
        shp = self.factor_shape(ell)
        num = torch.empty(shp, dtype=torch.float32, device=Y.device)
        den = torch.empty(shp, dtype=torch.float32, device=Y.device)
        nef_num_den_ex(self.h, ell, Y, mask, spec, factors, num, den, self.workspace(Y.device), stream)
        return num, den

    def loss_ex(self, Y, mask, spec, factors, stream=None):
        return nef_loss_ex(self.h, Y, mask, spec, factors, self.workspace(Y.device), stream)
