"""Thin ctypes binding of libffsat.so (include/ffsat.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels.  If the library is
missing this module raises at import-use time -- there is no CPU fallback.  Function
names mirror the C-ABI (ffsat_load, ffsat_eval, ...); `Context` / `Search` wrap them.

Buffers: numpy arrays are host buffers (on_device = 0, the library stages and
synchronises); torch CUDA tensors are device buffers (on_device = 1) and work is
enqueued on torch's current stream of that device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libffsat.so")

OR, XOR, XNOR, CARD_GE, CARD_LE, NAE = 0, 1, 2, 3, 4, 5
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_PARSE", 3: "ERR_RANGE", 4: "ERR_DUPVAR", 5: "ERR_BOUND",
          6: "ERR_NONFINITE", 7: "ERR_CUDA", 8: "ERR_NCCL", 9: "ERR_OOM"}
POLICY = {"ROF": 0, "RF": 1, "R": 2}


class FfsatError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ffsat_formula(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("n_cons", C.c_int64), ("kind", C.c_void_p), ("bound", C.c_void_p),
                ("weight", C.c_void_p), ("offsets", C.c_void_p), ("lits", C.c_void_p)]


class ffsat_options(C.Structure):
    _fields_ = [("precision", C.c_int32), ("device", C.c_int32), ("path", C.c_int32), ("batch_ref", C.c_int32)]


class ffsat_info_t(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("precision", C.c_int32), ("n_cons", C.c_int64), ("n_lits", C.c_int64),
                ("n_fast_cons", C.c_int64), ("n_sym_cons", C.c_int64), ("n_fast_lits", C.c_int64),
                ("n_sym_lits", C.c_int64), ("sym_root_lits", C.c_int64), ("path", C.c_int32), ("wide", C.c_int32),
                ("max_k", C.c_int32), ("pad", C.c_int32), ("device_bytes", C.c_int64), ("n_own_lits", C.c_int64),
                ("n_tree_cons", C.c_int64), ("tree_work", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ffsat_solve_params(C.Structure):
    _fields_ = [("eta0", C.c_double), ("eta_min", C.c_double), ("armijo_c1", C.c_double), ("alpha", C.c_double),
                ("max_inner", C.c_int32), ("check_every", C.c_int32), ("policy", C.c_int32),
                ("adaptive_weights", C.c_int32), ("timeout_s", C.c_double), ("accel", C.c_int32),
                ("reserved", C.c_int32)]


class ffsat_search_stats(C.Structure):
    _fields_ = [("round", C.c_int64), ("iterations", C.c_int64), ("active", C.c_int64), ("solved_point", C.c_int64),
                ("best_unsat", C.c_int64), ("best_point", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ffsat_search_buffers(C.Structure):
    _fields_ = [("x", C.c_void_p), ("grad", C.c_void_p), ("f", C.c_void_p), ("eta", C.c_void_p),
                ("unsat", C.c_void_p), ("U", C.c_void_p), ("weights", C.c_void_p), ("keys", C.c_void_p),
                ("solved", C.c_void_p), ("xp", C.c_void_p), ("x_prev", C.c_void_p), ("y", C.c_void_p),
                ("f_y", C.c_void_p), ("t", C.c_void_p), ("phase", C.c_void_p)]


class ffsat_result(C.Structure):
    _fields_ = [("sat", C.c_int32), ("reserved", C.c_int32), ("restarts", C.c_int64), ("iterations", C.c_int64),
                ("best_unsat", C.c_int64), ("best_falsified_weight", C.c_double), ("seconds", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


EXPORTS = ["ffsat_load", "ffsat_load_file", "ffsat_info", "ffsat_export", "ffsat_eval", "ffsat_set_weights",
           "ffsat_get_weights", "ffsat_check", "ffsat_search_create", "ffsat_search_set_x", "ffsat_search_begin_round",
           "ffsat_search_iterate", "ffsat_search_check", "ffsat_search_reduce", "ffsat_search_restart", "ffsat_search_stats_get",
           "ffsat_search_get_buffers", "ffsat_search_assignment", "ffsat_search_free", "ffsat_solve",
           "ffsat_default_params", "ffsat_last_error", "ffsat_version", "ffsat_free", "ffsat_launch_count",
           "ffsat_eval_profiled", "ffsat_layout_units"]

_lib = None


def lib():
    """Load libffsat.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libffsat.so not built ({LIB_PATH}); run __graft_entry__.build() -- there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "ffsat_load": ([C.POINTER(ffsat_formula), C.POINTER(ffsat_options), C.POINTER(P)], C.c_int),
        "ffsat_load_file": ([C.c_char_p, C.POINTER(ffsat_options), C.POINTER(P)], C.c_int),
        "ffsat_info": ([P, C.POINTER(ffsat_info_t)], C.c_int),
        "ffsat_export": ([P, P, P, P, P, P], C.c_int),
        "ffsat_eval": ([P, P, I64, I32, P, P, P, P], C.c_int),
        "ffsat_set_weights": ([P, P, I32, P], C.c_int),
        "ffsat_get_weights": ([P, P, I32, P], C.c_int),
        "ffsat_check": ([P, P, C.POINTER(I64), C.POINTER(C.c_double)], C.c_int),
        "ffsat_search_create": ([P, I64, I64, U64, C.POINTER(ffsat_solve_params), C.POINTER(P)], C.c_int),
        "ffsat_search_set_x": ([P, P, I32, P], C.c_int),
        "ffsat_search_begin_round": ([P, P], C.c_int),
        "ffsat_search_iterate": ([P, I32, P], C.c_int),
        "ffsat_search_check": ([P, P], C.c_int),
        "ffsat_search_reduce": ([P, P], C.c_int),
        "ffsat_search_restart": ([P, P, P], C.c_int),
        "ffsat_search_stats_get": ([P, P, C.POINTER(ffsat_search_stats)], C.c_int),
        "ffsat_search_get_buffers": ([P, C.POINTER(ffsat_search_buffers)], C.c_int),
        "ffsat_search_assignment": ([P, I64, P], C.c_int),
        "ffsat_search_free": ([P], None),
        "ffsat_solve": ([P, I64, I64, U64, C.POINTER(ffsat_solve_params), P, C.POINTER(ffsat_result)], C.c_int),
        "ffsat_default_params": ([C.POINTER(ffsat_solve_params)], None),
        "ffsat_last_error": ([P], C.c_char_p),
        "ffsat_version": ([], C.c_char_p),
        "ffsat_free": ([P], None),
        "ffsat_launch_count": ([P, C.POINTER(I64)], C.c_int),
        "ffsat_eval_profiled": ([P, P, I64, P, P, P, P, C.POINTER(C.c_double)], C.c_int),
        "ffsat_layout_units": ([P, C.POINTER(I64), P, I64, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(status, ctx_ptr=None):
    if status != 0:
        msg = lib().ffsat_last_error(ctx_ptr)
        raise FfsatError(status, msg.decode() if msg else "")


# ----------------------------------------------------------------------------- marshalling helpers

def _is_torch(t):
    return type(t).__module__.startswith("torch")


def _buf(a):
    """(pointer, on_device) for a numpy array or torch tensor (None -> null)."""
    if a is None:
        return None, None
    if _is_torch(a):
        assert a.is_contiguous(), "tensors must be contiguous"
        return C.c_void_p(a.data_ptr()), bool(a.is_cuda)
    assert isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous numpy arrays"
    return a.ctypes.data_as(C.c_void_p), False


def _stream(stream, like=None):
    if stream is not None:
        return C.c_void_p(int(stream))
    if like is not None and _is_torch(like) and like.is_cuda:
        import torch
        return C.c_void_p(torch.cuda.current_stream(like.device).cuda_stream)
    return C.c_void_p(0)


# ----------------------------------------------------------------------------- C-ABI mirrors

def ffsat_load(n_vars, kind, bound, weight, offsets, lits, precision=0, device=0, path=0, batch_ref=0):
    kind = np.ascontiguousarray(kind, np.uint8)
    m = len(kind)
    bound = np.ascontiguousarray(bound if bound is not None else np.zeros(m), np.int32)
    weight = np.ascontiguousarray(weight if weight is not None else np.ones(m), np.float64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    lits = np.ascontiguousarray(lits, np.int32)
    f = ffsat_formula(int(n_vars), m, kind.ctypes.data, bound.ctypes.data, weight.ctypes.data, offsets.ctypes.data,
                      lits.ctypes.data)
    o = ffsat_options(int(precision), int(device), int(path), int(batch_ref))
    out = C.c_void_p()
    _check(lib().ffsat_load(C.byref(f), C.byref(o), C.byref(out)))
    return out


def ffsat_load_file(path, precision=0, device=0, opt_path=0, batch_ref=0):
    o = ffsat_options(int(precision), int(device), int(opt_path), int(batch_ref))
    out = C.c_void_p()
    _check(lib().ffsat_load_file(str(path).encode(), C.byref(o), C.byref(out)))
    return out


def ffsat_info(ctx):
    i = ffsat_info_t()
    _check(lib().ffsat_info(ctx, C.byref(i)), ctx)
    return i.as_dict()


def ffsat_eval(ctx, x, B, f_out, grad_out=None, unsat_out=None, stream=None):
    px, dev = _buf(x)
    pf, _ = _buf(f_out)
    pg, _ = _buf(grad_out)
    pu, _ = _buf(unsat_out)
    _check(lib().ffsat_eval(ctx, px, int(B), int(dev), pf, pg, pu, _stream(stream, x)), ctx)


def ffsat_check(ctx, assignment):
    a = np.ascontiguousarray(assignment, np.int8)
    n = C.c_int64()
    w = C.c_double()
    _check(lib().ffsat_check(ctx, a.ctypes.data_as(C.c_void_p), C.byref(n), C.byref(w)), ctx)
    return int(n.value), float(w.value)


def ffsat_default_params(**kw):
    p = ffsat_solve_params()
    lib().ffsat_default_params(C.byref(p))
    for k, v in kw.items():
        if k == "policy" and isinstance(v, str):
            v = POLICY[v]
        setattr(p, k, v)
    return p


def ffsat_free(ctx):
    lib().ffsat_free(ctx)


def ffsat_version():
    return lib().ffsat_version().decode()


# ----------------------------------------------------------------------------- convenience wrappers

class Context:
    """A loaded formula on one device (or device=-1: host-only, parse/validate/check)."""

    def __init__(self, ptr, keep=None):
        self.ptr = ptr
        self.info = ffsat_info(ptr)
        self.n = self.info["n_vars"]
        self.m = self.info["n_cons"]
        self.dtype = np.float64 if self.info["precision"] == 64 else np.float32

    @classmethod
    def from_arrays(cls, n, kind, bound, weight, offsets, lits, precision=0, device=0, path=0, batch_ref=0):
        return cls(ffsat_load(n, kind, bound, weight, offsets, lits, precision, device, path, batch_ref))

    @classmethod
    def from_instance(cls, inst, **kw):
        return cls.from_arrays(inst.n, inst.kind, inst.bound, inst.weight, inst.offsets, inst.lits, **kw)

    @classmethod
    def from_file(cls, path, precision=0, device=0, opt_path=0, batch_ref=0):
        return cls(ffsat_load_file(path, precision, device, opt_path, batch_ref))

    def close(self):
        if self.ptr:
            ffsat_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self):
        m, L = self.m, self.info["n_lits"]
        kind = np.zeros(m, np.uint8); bound = np.zeros(m, np.int32); w = np.zeros(m)
        off = np.zeros(m + 1, np.int64); lits = np.zeros(L, np.int32)
        _check(lib().ffsat_export(self.ptr, kind.ctypes.data, bound.ctypes.data, w.ctypes.data, off.ctypes.data,
                                  lits.ctypes.data), self.ptr)
        return kind, bound, w, off, lits

    def eval(self, x, grad=True, unsat=False, stream=None):
        """f, grad, unsat at points x [B][n] (numpy -> host path; torch CUDA tensor -> device path)."""
        if _is_torch(x) and x.is_cuda:
            import torch
            B = x.shape[0]
            f = torch.empty(B, dtype=torch.float64, device=x.device)
            g = torch.empty_like(x) if grad else None
            u = torch.empty(B, dtype=torch.int32, device=x.device) if unsat else None
            ffsat_eval(self.ptr, x, B, f, g, u, stream)
            return f, g, u
        x = np.ascontiguousarray(np.atleast_2d(x), self.dtype)
        B = x.shape[0]
        f = np.zeros(B)
        g = np.zeros_like(x) if grad else None
        u = np.zeros(B, np.int32) if unsat else None
        ffsat_eval(self.ptr, x, B, f, g, u, stream)
        return f, g, u

    def layout_units(self):
        """(units [U][4] = bucket, count, first position, tiled flag; order [m] position -> input constraint)."""
        nu = C.c_int64()
        _check(lib().ffsat_layout_units(self.ptr, C.byref(nu), None, 0, None), self.ptr)
        units = np.zeros((nu.value, 4), np.int64)
        order = np.zeros(self.m, np.int64)
        _check(lib().ffsat_layout_units(self.ptr, C.byref(nu), units.ctypes.data_as(C.c_void_p), nu.value,
                                        order.ctypes.data_as(C.c_void_p)), self.ptr)
        return units, order

    def order(self):
        """Position -> input-constraint map of the library's internal constraint order (per-constraint device arrays
        such as a search's U and weights are in position order: input[order[p]] = position[p])."""
        return self.layout_units()[1]

    def to_input_order(self, a):
        """A per-constraint array in position order -> input order."""
        a = np.asarray(a)
        out = np.empty_like(a)
        out[self.order()] = a
        return out

    def launch_count(self):
        n = C.c_int64()
        _check(lib().ffsat_launch_count(self.ptr, C.byref(n)), self.ptr)
        return int(n.value)

    def eval_profiled(self, x, f, g=None, u=None, stream=None):
        """Device eval with per-phase CUDA-event times (ms): fast kernel, root kernels, grad reduce, f reduce."""
        ms = (C.c_double * 4)()
        px, dev = _buf(x)
        assert dev, "eval_profiled needs device tensors"
        _check(lib().ffsat_eval_profiled(self.ptr, px, int(x.shape[0]), _buf(f)[0], _buf(g)[0], _buf(u)[0],
                                         _stream(stream, x), ms), self.ptr)
        return list(ms)

    def set_weights(self, w, stream=None):
        if _is_torch(w):
            pw, dev = _buf(w)
            _check(lib().ffsat_set_weights(self.ptr, pw, int(dev), _stream(stream, w)), self.ptr)
        else:
            w = np.ascontiguousarray(w, np.float64)
            _check(lib().ffsat_set_weights(self.ptr, w.ctypes.data_as(C.c_void_p), 0, _stream(stream)), self.ptr)

    def get_weights(self):
        w = np.zeros(self.m)
        _check(lib().ffsat_get_weights(self.ptr, w.ctypes.data_as(C.c_void_p), 0, C.c_void_p(0)), self.ptr)
        return w

    def check(self, assignment):
        return ffsat_check(self.ptr, assignment)

    def solve(self, batch, max_restarts, seed=0, **params):
        p = ffsat_default_params(**params)
        a = np.zeros(self.n, np.int8)
        r = ffsat_result()
        _check(lib().ffsat_solve(self.ptr, int(batch), int(max_restarts), int(seed), C.byref(p),
                                 a.ctypes.data_as(C.c_void_p), C.byref(r)), self.ptr)
        return r.as_dict(), a

    def search(self, batch, seed=0, point0=0, **params):
        return Search(self, batch, seed, point0, **params)


class Search:
    """Device-resident batched CLS state (Alg. 1 with p_t = batch)."""

    def __init__(self, ctx: Context, batch, seed=0, point0=0, **params):
        self.ctx = ctx
        self.B = int(batch)
        self.point0 = int(point0)
        self.params = ffsat_default_params(**params)
        self.ptr = C.c_void_p()
        _check(lib().ffsat_search_create(ctx.ptr, self.B, self.point0, int(seed), C.byref(self.params),
                                         C.byref(self.ptr)), ctx.ptr)

    def close(self):
        if self.ptr:
            lib().ffsat_search_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_x(self, x, stream=None):
        px, dev = _buf(x)
        _check(lib().ffsat_search_set_x(self.ptr, px, int(dev), _stream(stream, x)), self.ctx.ptr)

    def begin_round(self, stream=None):
        _check(lib().ffsat_search_begin_round(self.ptr, _stream(stream)), self.ctx.ptr)

    def iterate(self, n, stream=None):
        _check(lib().ffsat_search_iterate(self.ptr, int(n), _stream(stream)), self.ctx.ptr)

    def check(self, stream=None):
        _check(lib().ffsat_search_check(self.ptr, _stream(stream)), self.ctx.ptr)

    def reduce(self, stream=None):
        """Device-side any-solved / incumbent keys into tensors()['keys'] (asynchronous)."""
        _check(lib().ffsat_search_reduce(self.ptr, _stream(stream)), self.ctx.ptr)

    def restart(self, U_global=None, stream=None):
        pU = C.c_void_p(U_global.data_ptr()) if U_global is not None else None
        _check(lib().ffsat_search_restart(self.ptr, pU, _stream(stream)), self.ctx.ptr)

    def stats(self, stream=None):
        s = ffsat_search_stats()
        _check(lib().ffsat_search_stats_get(self.ptr, _stream(stream), C.byref(s)), self.ctx.ptr)
        return s.as_dict()

    def buffers(self):
        b = ffsat_search_buffers()
        _check(lib().ffsat_search_get_buffers(self.ptr, C.byref(b)), self.ctx.ptr)
        return b

    def assignment(self, local_point):
        a = np.zeros(self.ctx.n, np.int8)
        _check(lib().ffsat_search_assignment(self.ptr, int(local_point), a.ctypes.data_as(C.c_void_p)), self.ctx.ptr)
        return a

    def tensors(self):
        """torch views of the device buffers (x, grad, f, eta, unsat, U, weights, keys, solved, xp; in FISTA mode also
        x_prev, y, f_y, t, phase -- grad is then the gradient at y); U and weights are in
        the library's position order (Context.order() maps position -> input constraint)."""
        import torch
        b = self.buffers()
        n, m, B = self.ctx.n, self.ctx.m, self.B
        tdt = torch.float64 if self.ctx.dtype == np.float64 else torch.float32
        dev = torch.device("cuda", torch.cuda.current_device())

        def view(ptr, count, dtype):
            return _device_view(ptr, count, dtype, dev)
        out = {"x": view(b.x, B * n, tdt).view(B, n), "grad": view(b.grad, B * n, tdt).view(B, n),
                "f": view(b.f, B, torch.float64), "eta": view(b.eta, B, torch.float64),
                "unsat": view(b.unsat, B, torch.int32), "U": view(b.U, m, torch.int32),
                "weights": view(b.weights, m, tdt), "keys": view(b.keys, 2, torch.int64),
                "solved": view(b.solved, B, torch.int32), "xp": view(b.xp, B * n, tdt).view(B, n)}
        if b.y:   # FISTA state (accel = 1)
            out.update({"x_prev": view(b.x_prev, B * n, tdt).view(B, n), "y": view(b.y, B * n, tdt).view(B, n),
                        "f_y": view(b.f_y, B, torch.float64), "t": view(b.t, B, torch.float64),
                        "phase": view(b.phase, B, torch.int32)})
        return out


def _device_view(ptr, count, dtype, device):
    """Zero-copy torch view of library-owned device memory (lifetime tied to the owner object)."""
    import torch

    class _CAI:
        def __init__(self):
            typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8"}[dtype]
            self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                             "data": (int(ptr or 0), False), "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=device)
