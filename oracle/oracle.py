"""ctypes binding of the CPU oracle (oracle/rocp_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
timed CPU baseline.  The product (paper_2007_10798_b200) never imports it.

All arrays are numpy; matrices are column-major (Fortran order), matching the
reference's Eigen::MatrixXd layout (tensor.hpp:10).  Tensors are flat float64
arrays, first index fastest (tensor.hpp:14-16).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "librocp_oracle.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class DomainError(OracleError):
    pass


class NumericalError(OracleError):
    def __init__(self, code, msg, sweep=None):
        super().__init__(code, msg)
        self.sweep = sweep


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_codomain_size.restype = C.c_int64
        _lib.orc_auto_sample_count.restype = C.c_int64
        _lib.orc_stream_t_len.restype = C.c_int64
        _lib.orc_stream_new.argtypes = [C.c_int, _i64p, C.c_int, C.c_int64, C.c_int,
                                        C.POINTER(_f64p), C.c_int64, C.POINTER(_f64p), C.c_int,
                                        C.POINTER(C.c_void_p)]
        _lib.orc_stream_free.argtypes = [C.c_void_p]
        _lib.orc_stream_consume.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_uint64, C.c_uint32]
        _lib.orc_stream_last_residuals.argtypes = [C.c_void_p, _f64p]
        _lib.orc_stream_consume_sharded.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_uint64, C.c_uint32,
                                                    C.c_int]
        _lib.orc_stream_update_last_mode_with.argtypes = [C.c_void_p, _f64p, C.c_int64, _i64p,
                                                          C.c_int64, _f64p, _f64p,
                                                          C.POINTER(C.c_int)]
        _lib.orc_stream_append_temporal.argtypes = [C.c_void_p, _f64p, C.c_int64]
        _lib.orc_stream_update_mode_with.argtypes = [C.c_void_p, _f64p, C.c_int64, _f64p, C.c_int,
                                                     _i64p, C.c_int64, _f64p, _f64p,
                                                     C.POINTER(C.c_int)]
        _lib.orc_stream_finish_batch.argtypes = [C.c_void_p, C.c_int64]
        _lib.orc_stream_get.argtypes = [C.c_void_p, C.c_int, C.c_int, _f64p]
        _lib.orc_stream_set.argtypes = [C.c_void_p, C.c_int, C.c_int, _f64p]
        _lib.orc_stream_t_len.argtypes = [C.c_void_p]
        _lib.orc_stream_regularized.argtypes = [C.c_void_p]
        _lib.orc_draw_samples.argtypes = [_i64p, C.c_int, C.c_int, C.c_int64, C.c_uint64,
                                          C.c_uint32, C.c_uint32, _i64p, _i64p]
        _lib.orc_cprand.argtypes = [_f64p, _i64p, C.c_int, C.c_int, C.c_int64, C.c_double, C.c_int,
                                    C.c_uint64, C.POINTER(_f64p), C.POINTER(_f64p), _f64p,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    _f64p]
    return _lib


def _p(a, t=_f64p):
    return a.ctypes.data_as(t)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.asfortranarray(a, dtype=np.float64)


def _check(rc, sweep=None):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise DomainError(rc, msg)
    if rc == 2:
        raise NumericalError(rc, msg, sweep)
    raise OracleError(rc, msg)


def _ptr_array(mats):
    arr = (_f64p * len(mats))()
    for k, m in enumerate(mats):
        arr[k] = m.ctypes.data_as(_f64p)
    return arr


# ---- RNG / index map ---------------------------------------------------------
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(out, _u32p))
    return [int(x) for x in out]


def codomain_size(dims, mode):
    d = _i64(dims)
    return int(lib().orc_codomain_size(_p(d, _i64p), len(d), mode))


def linear_index(multi, dims, mode):
    d, m = _i64(dims), _i64(multi)
    j = C.c_int64(0)
    _check(lib().orc_linear_index(_p(m, _i64p), _p(d, _i64p), len(d), mode, C.byref(j)))
    return j.value


def decode_index(j, dims, mode):
    d = _i64(dims)
    out = np.zeros(len(d) - 1, dtype=np.int64)
    _check(lib().orc_decode_index(C.c_int64(j), _p(d, _i64p), len(d), mode, _p(out, _i64p)))
    return [int(x) for x in out]


def auto_sample_count(rank):
    v = int(lib().orc_auto_sample_count(rank))
    if v < 0:
        raise DomainError(1, "rank must be positive")
    return v


def from_rows(dims, mode, rows):
    d, r = _i64(dims), _i64(rows)
    dec = np.zeros(len(r) * (len(d) - 1), dtype=np.int64)
    _check(lib().orc_from_rows(_p(d, _i64p), len(d), mode, _p(r, _i64p), C.c_int64(len(r)),
                               _p(dec, _i64p)))
    return dec.reshape(len(r), len(d) - 1)


def draw_samples(dims, mode, s, seed, batch, iteration):
    d = _i64(dims)
    rows = np.zeros(max(s, 0), dtype=np.int64)
    dec = np.zeros(max(s, 0) * (len(d) - 1), dtype=np.int64)
    _check(lib().orc_draw_samples(_p(d, _i64p), len(d), mode, s, seed, batch, iteration,
                                  _p(rows, _i64p), _p(dec, _i64p)))
    return rows, dec.reshape(max(s, 0), len(d) - 1)


# ---- sampling primitives -----------------------------------------------------
def sample_unfolding(t, dims, mode, decoded):
    t = np.ascontiguousarray(t, dtype=np.float64).ravel(order="K")
    d, dec = _i64(dims), _i64(decoded)
    s = dec.shape[0]
    out = np.zeros((dims[mode - 1], s), dtype=np.float64, order="F")
    _check(lib().orc_sample_unfolding(_p(t), _p(d, _i64p), len(d), mode, _p(dec, _i64p),
                                      C.c_int64(s), _p(out)))
    return out


def sampled_khatri_rao(decoded, factors):
    """factors in factors_excluding order (kruskal.cpp:44-53)."""
    dec = _i64(decoded)
    s = dec.shape[0]
    fs = [_f64(f) for f in factors]
    rank = fs[0].shape[1]
    rows = _i64([f.shape[0] for f in fs])
    z = np.zeros((s, rank), dtype=np.float64, order="F")
    _check(lib().orc_sampled_khatri_rao(_p(dec, _i64p), C.c_int64(s), len(fs), _ptr_array(fs),
                                        _p(rows, _i64p), rank, _p(z)))
    return z


def gram(z):
    z = _f64(z)
    g = np.zeros((z.shape[1], z.shape[1]), order="F")
    lib().orc_gram(_p(z), C.c_int64(z.shape[0]), z.shape[1], _p(g))
    return g


def contract(x, z):
    x, z = _f64(x), _f64(z)
    out = np.zeros((x.shape[0], z.shape[1]), order="F")
    lib().orc_contract(_p(x), C.c_int64(x.shape[0]), C.c_int64(x.shape[1]), _p(z), z.shape[1],
                       _p(out))
    return out


def solve_gram(g, rhs):
    g, rhs = _f64(g), _f64(rhs)
    out = np.zeros(rhs.shape, order="F")
    reg = C.c_int(0)
    _check(lib().orc_solve_gram(_p(g), _p(rhs), C.c_int64(rhs.shape[0]), g.shape[0], _p(out),
                                C.byref(reg)))
    return out, bool(reg.value)


def gram_decision(g):
    """solve_gram's regularisation decision (solve.cpp:17-33) in canonical form:
    (mode, regularized, path, jacobi_lo, jacobi_hi); mode 0 = zero solution, path 0/1 =
    settled by the certificate (no-reg / reg), 2 = exact Jacobi eigenvalues."""
    g = _f64(g)
    mode, reg, path = C.c_int(0), C.c_int(0), C.c_int(0)
    lo, hi = C.c_double(0.0), C.c_double(0.0)
    _check(lib().orc_gram_decision(_p(g), g.shape[0], C.byref(mode), C.byref(reg), C.byref(path),
                                   C.byref(lo), C.byref(hi)))
    return mode.value, bool(reg.value), path.value, lo.value, hi.value


def solve_sampled_ls(z, x):
    z, x = _f64(z), _f64(x)
    if x.shape[1] != z.shape[0]:
        raise DomainError(1, "solve_sampled_ls: sample counts of z_s and x_s differ")
    out = np.zeros((x.shape[0], z.shape[1]), order="F")
    reg, und = C.c_int(0), C.c_int(0)
    _check(lib().orc_solve_sampled_ls(_p(z), _p(x), C.c_int64(z.shape[0]), C.c_int64(x.shape[0]),
                                      z.shape[1], _p(out), C.byref(reg), C.byref(und)))
    return out, bool(reg.value), bool(und.value)


# ---- model -------------------------------------------------------------------
def model_fitness(t, dims, factors):
    t = np.ascontiguousarray(t, dtype=np.float64).ravel(order="K")
    d = _i64(dims)
    fs = [_f64(f) for f in factors]
    fit = C.c_double(0)
    _check(lib().orc_model_fitness(_p(t), _p(d, _i64p), len(d), _ptr_array(fs), fs[0].shape[1],
                                   C.byref(fit)))
    return fit.value


def reconstruct(factors, dims):
    d = _i64(dims)
    fs = [_f64(f) for f in factors]
    out = np.zeros(int(np.prod(dims)), dtype=np.float64)
    _check(lib().orc_reconstruct(_ptr_array(fs), _p(d, _i64p), len(d), fs[0].shape[1], _p(out)))
    return out


def khatri_rao(a, b):
    a, b = _f64(a), _f64(b)
    out = np.zeros((a.shape[0] * b.shape[0], a.shape[1]), order="F")
    lib().orc_khatri_rao(_p(a), C.c_int64(a.shape[0]), _p(b), C.c_int64(b.shape[0]), a.shape[1],
                         _p(out))
    return out


def khatri_rao_list(ms):
    acc = _f64(ms[0])
    for m in ms[1:]:
        acc = khatri_rao(acc, m)
    return acc


def factors_excluding(factors, mode):
    return [factors[k - 1] for k in range(len(factors), 0, -1) if k != mode]


# ---- cprand ------------------------------------------------------------------
class InitResult:
    def __init__(self, model, best_sampled_kr, best_fitness, iterations, regularized, fit_trace):
        self.model = model
        self.best_sampled_kr = best_sampled_kr
        self.best_sampled_factors = [model[n] for n in range(len(model) - 1)]
        self.best_fitness = best_fitness
        self.iterations = iterations
        self.regularized = regularized
        self.fit_trace = fit_trace


def cprand_decompose(t, dims, rank, init_factors, seed, samples=0, tol=1e-4, max_iters=100):
    t = np.ascontiguousarray(t, dtype=np.float64).ravel(order="K")
    d = _i64(dims)
    N = len(dims)
    fs = [np.array(f, dtype=np.float64, order="F", copy=True) for f in init_factors]
    s = samples if samples > 0 else auto_sample_count(rank)
    kr = [np.zeros((s, rank), order="F") for _ in range(N - 1)]
    best, iters, reg, errs = C.c_double(0), C.c_int(0), C.c_int(0), C.c_int(0)
    trace = np.zeros(max(max_iters, 1), dtype=np.float64)
    rc = lib().orc_cprand(_p(t), _p(d, _i64p), N, rank, samples, tol, max_iters, seed,
                          _ptr_array(fs), _ptr_array(kr) if N > 1 else None, C.byref(best),
                          C.byref(iters), C.byref(reg), C.byref(errs), _p(trace))
    _check(rc, sweep=errs.value)
    return InitResult(fs, kr, best.value, iters.value, bool(reg.value), trace[: iters.value])


# ---- stream ------------------------------------------------------------------
class Stream:
    """RocpStream restatement (rocp.hpp:85-107) with counter-RNG draws."""

    def __init__(self, init_factors, t_init, best_sampled_kr, s, literal_init=False,
                 regularized=False):
        self.order = len(init_factors)
        self.rank = init_factors[0].shape[1]
        self.head = [f.shape[0] for f in init_factors[:-1]]
        self.s = s
        fs = [_f64(f) for f in init_factors]
        kr = [_f64(z) for z in best_sampled_kr]
        for z in kr:
            if z.shape[0] != s:
                raise DomainError(1, "init_state: sampled Khatri-Rao row count differs from s")
        hd = _i64(self.head)
        h = C.c_void_p()
        _check(lib().orc_stream_new(self.order, _p(hd, _i64p), self.rank, s, int(literal_init),
                                    _ptr_array(fs), t_init, _ptr_array(kr), int(regularized),
                                    C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_stream_free(self._h)
            self._h = None

    def _slab(self, x_new, batch):
        x = np.ascontiguousarray(x_new, dtype=np.float64).ravel(order="K")
        if x.size != int(np.prod(self.head)) * batch:
            raise DomainError(1, "batch head extents do not match stream")
        return x

    def consume(self, x_new, batch, seed, batch_id):
        x = self._slab(x_new, batch)
        _check(lib().orc_stream_consume(self._h, _p(x), batch, seed, batch_id))

    def consume_sharded(self, x_new, batch, seed, batch_id, virtual_shards):
        """Mode-1 sharded consume, canonical order of `virtual_shards` row ranges."""
        x = self._slab(x_new, batch)
        _check(lib().orc_stream_consume_sharded(self._h, _p(x), batch, seed, batch_id, virtual_shards))

    def last_residuals(self):
        out = np.zeros(self.order)
        _check(lib().orc_stream_last_residuals(self._h, _p(out)))
        return out

    def update_last_mode_with(self, x_new, batch, rows):
        x = self._slab(x_new, batch)
        r = _i64(rows)
        u = np.zeros((batch, self.rank), order="F")
        z = np.zeros((len(r), self.rank), order="F")
        reg = C.c_int(0)
        _check(lib().orc_stream_update_last_mode_with(self._h, _p(x), batch, _p(r, _i64p), len(r),
                                                      _p(u), _p(z), C.byref(reg)))
        return u, z, bool(reg.value)

    def append_temporal(self, u_new):
        u = _f64(u_new)
        _check(lib().orc_stream_append_temporal(self._h, _p(u), u.shape[0]))

    def update_mode_with(self, x_new, batch, u_new, mode, rows):
        x = self._slab(x_new, batch)
        r = _i64(rows)
        u = _f64(u_new)
        z = np.zeros((len(r), self.rank), order="F")
        I = self.head[mode - 1]
        xs = np.zeros((I, len(r)), order="F")
        reg = C.c_int(0)
        _check(lib().orc_stream_update_mode_with(self._h, _p(x), batch, _p(u), mode, _p(r, _i64p),
                                                 len(r), _p(z), _p(xs), C.byref(reg)))
        return z, xs, bool(reg.value)

    def finish_batch(self, batch):
        lib().orc_stream_finish_batch(self._h, batch)

    def factor(self, mode):
        out = np.zeros((self.head[mode - 1], self.rank), order="F")
        _check(lib().orc_stream_get(self._h, 0, mode, _p(out)))
        return out

    def p(self, mode):
        out = np.zeros((self.head[mode - 1], self.rank), order="F")
        _check(lib().orc_stream_get(self._h, 1, mode, _p(out)))
        return out

    def q(self, mode):
        out = np.zeros((self.rank, self.rank), order="F")
        _check(lib().orc_stream_get(self._h, 2, mode, _p(out)))
        return out

    def set(self, what, mode, arr):
        a = _f64(arr)
        _check(lib().orc_stream_set(self._h, what, mode, _p(a)))

    @property
    def t_len(self):
        return int(lib().orc_stream_t_len(self._h))

    @property
    def regularized(self):
        return bool(lib().orc_stream_regularized(self._h))

    def temporal(self):
        out = np.zeros((self.t_len, self.rank), order="F")
        _check(lib().orc_stream_get(self._h, 3, 0, _p(out)))
        return out

    def model(self):
        return [self.factor(n) for n in range(1, self.order)] + [self.temporal()]


def online_full_init(x, dims, factors):
    d = _i64(dims)
    x = np.ascontiguousarray(x, dtype=np.float64).ravel(order="K")
    fs = [_f64(f) for f in factors]
    R = fs[0].shape[1]
    p = [np.zeros((dims[n], R), order="F") for n in range(len(dims) - 1)]
    q = [np.zeros((R, R), order="F") for _ in range(len(dims) - 1)]
    _check(lib().orc_online_full_init(_p(x), _p(d, _i64p), len(d), _ptr_array(fs), R,
                                      _ptr_array(p), _ptr_array(q)))
    return p, q


def online_full_update(x_new, dims, head_factors, p, q):
    """Mutates head_factors, p, q in place (Fortran arrays); returns u_new."""
    d = _i64(dims)
    x = np.ascontiguousarray(x_new, dtype=np.float64).ravel(order="K")
    R = head_factors[0].shape[1]
    u = np.zeros((dims[-1], R), order="F")
    _check(lib().orc_online_full_update(_p(x), _p(d, _i64p), len(d), _ptr_array(head_factors), R,
                                        _ptr_array(p), _ptr_array(q), _p(u)))
    return u
