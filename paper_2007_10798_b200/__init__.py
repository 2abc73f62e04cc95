"""B200-native ROCP hot path (randomized online CP decomposition, arXiv 2007.10798).

The product is librocp_b200.so (CUDA, sm_100a) behind the C ABI in
include/rocp_b200.h.  This module is a thin Python host mirror of the
reference's C++ API (reference proj/include/rocp/*.hpp) over that ABI, used by
the tests and bench.py.  There is no CPU fallback: if the shared library is
missing or no GPU is present, calls fail loudly.

Reference interfaces mirrored (file:line in /root/reference/proj):
  draw_samples / sample_unfolding / sampled_khatri_rao   sampling.hpp:35-48
  solve_gram / solve_sampled_ls                          solve.hpp:17-24
  model_fitness                                          kruskal.hpp:38-39
  cprand_decompose -> InitResult                         cprand.hpp:19-37
  RocpStream (consume, model, state)                     rocp.hpp:85-107
  update_last_mode_with / update_mode_with (replay)      rocp.hpp:52-75
Matrices are numpy column-major (Fortran) arrays, like Eigen::MatrixXd.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import subprocess
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ROCP_B200_LIB") or os.path.join(_HERE, "_lib", "librocp_b200.so")  # override: profiling builds

# status codes (include/rocp_b200.h)
OK, E_DOMAIN, E_NUMERICAL, E_CUDA, E_NCCL, E_OOM, E_STATE, E_IO = range(8)

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p

# Every symbol declared in include/rocp_b200.h: (name, restype, argtypes).
SIGNATURES = [
    ("rocp_create", C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_vp)]),
    ("rocp_create_emulated_rank", C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    ("rocp_emulated_group_consume_range", C.c_int, [C.POINTER(_vp), C.c_int, C.POINTER(_vp), C.c_int64, C.c_int64,
                                                    C.c_int64, C.c_uint64, C.c_uint32]),
    ("rocp_destroy", None, [_vp]),
    ("rocp_last_error", C.c_char_p, [_vp]),
    ("rocp_set_gather_sms", C.c_int, [_vp, C.c_int]),
    ("rocp_set_chain_sms", C.c_int, [_vp, C.c_int]),
    ("rocp_sm_count", C.c_int, [_vp, C.POINTER(C.c_int)]),
    ("rocp_synchronize", C.c_int, [_vp]),
    ("rocp_kernel_launches", C.c_uint64, [_vp]),
    ("rocp_nccl_id_size", C.c_int, []),
    ("rocp_nccl_get_unique_id", C.c_int, [_vp]),
    ("rocp_tensor_create", C.c_int, [_vp, _i64p, C.c_int, _f64p, C.POINTER(_vp)]),
    ("rocp_tensor_slab", C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.POINTER(_vp)]),
    ("rocp_tensor_rows", C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.POINTER(_vp)]),
    ("rocp_tensor_write_file", C.c_int, [_vp, _vp, C.c_char_p]),
    ("rocp_tensor_read_file", C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    ("rocp_tensor_free", None, [_vp]),
    ("rocp_tensor_upload", C.c_int, [_vp, _vp, _f64p]),
    ("rocp_tensor_download", C.c_int, [_vp, _vp, _f64p]),
    ("rocp_tensor_device_ptr", _vp, [_vp]),
    ("rocp_tensor_numel", C.c_int64, [_vp]),
    ("rocp_generate_synthetic", C.c_int, [_vp, _vp, C.POINTER(_f64p), C.c_int, C.c_int,
                                          C.c_double, C.c_uint64]),
    ("rocp_draw_samples", C.c_int, [_vp, _i64p, C.c_int, C.c_int, C.c_int64, C.c_uint64,
                                    C.c_uint32, C.c_uint32, _i64p, _i64p]),
    ("rocp_decode_rows", C.c_int, [_vp, _i64p, C.c_int, C.c_int, _i64p, C.c_int64, _i64p]),
    ("rocp_sample_unfolding", C.c_int, [_vp, _vp, C.c_int, _i64p, C.c_int64, _f64p]),
    ("rocp_sampled_khatri_rao", C.c_int, [_vp, _i64p, C.c_int64, C.c_int, C.POINTER(_f64p),
                                          _i64p, C.c_int, _f64p]),
    ("rocp_gram", C.c_int, [_vp, _f64p, C.c_int64, C.c_int, _f64p]),
    ("rocp_contract", C.c_int, [_vp, _f64p, C.c_int64, C.c_int64, _f64p, C.c_int, _f64p]),
    ("rocp_solve_gram", C.c_int, [_vp, _f64p, _f64p, C.c_int64, C.c_int, _f64p,
                                  C.POINTER(C.c_int)]),
    ("rocp_solve_sampled_ls", C.c_int, [_vp, _f64p, _f64p, C.c_int64, C.c_int64, C.c_int, _f64p,
                                        C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("rocp_model_fitness", C.c_int, [_vp, _vp, C.POINTER(_f64p), C.c_int, _f64p]),
    ("rocp_cprand", C.c_int, [_vp, _vp, C.c_int, C.c_int64, C.c_double, C.c_int, C.c_uint64,
                              C.POINTER(_f64p), C.POINTER(_f64p), _f64p, C.POINTER(C.c_int),
                              C.POINTER(C.c_int), C.POINTER(C.c_int), _f64p]),
    ("rocp_stream_create", C.c_int, [_vp, C.c_int, _i64p, C.c_int, C.c_int64, C.c_int,
                                     C.POINTER(_f64p), C.c_int64, C.POINTER(_f64p), C.c_int,
                                     C.c_int64, C.POINTER(_vp)]),
    ("rocp_stream_create_from_init", C.c_int, [_vp, C.c_int, C.c_int64, C.POINTER(_vp)]),
    ("rocp_stream_free", None, [_vp]),
    ("rocp_stream_shard", C.c_int, [_vp, C.c_int]),
    ("rocp_stream_write_state", C.c_int, [_vp, C.c_char_p]),
    ("rocp_stream_read_state", C.c_int, [_vp, C.c_char_p]),
    ("rocp_stream_write_checkpoint", C.c_int, [_vp, C.c_char_p]),
    ("rocp_stream_consume_file", C.c_int, [_vp, C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_uint32,
                                           C.c_int]),
    ("rocp_stream_create_from_checkpoint", C.c_int, [_vp, C.c_char_p, C.c_int64, C.POINTER(_vp)]),
    ("rocp_stream_shard_info", C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("rocp_stream_consume", C.c_int, [_vp, _vp, C.c_uint64, C.c_uint32]),
    ("rocp_stream_consume_host", C.c_int, [_vp, _f64p, C.c_int64, C.c_uint64, C.c_uint32]),
    ("rocp_stream_consume_range", C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                            C.c_uint32]),
    ("rocp_stream_consume_range_host", C.c_int, [_vp, _f64p, C.c_int64, C.c_int64, C.c_uint64, C.c_uint32,
                                                 C.c_int]),
    ("rocp_stream_update_last_mode_with", C.c_int, [_vp, _vp, _i64p, C.c_int64, _f64p, _f64p,
                                                    C.POINTER(C.c_int)]),
    ("rocp_stream_append_temporal", C.c_int, [_vp, _f64p, C.c_int64]),
    ("rocp_stream_update_mode_with", C.c_int, [_vp, _vp, _f64p, C.c_int, _i64p, C.c_int64, _f64p,
                                               _f64p, C.POINTER(C.c_int)]),
    ("rocp_stream_finish_batch", C.c_int, [_vp, C.c_int64]),
    ("rocp_probe_random_reads", C.c_int, [_vp, _vp, C.c_int64, C.c_uint64, C.POINTER(C.c_float)]),
    ("rocp_decision_stats", C.c_int, [_vp, C.POINTER(C.c_uint64), C.c_int]),
    ("rocp_stream_mark_regularized", C.c_int, [_vp]),
    ("rocp_stream_get", C.c_int, [_vp, C.c_int, C.c_int, _f64p]),
    ("rocp_stream_set", C.c_int, [_vp, C.c_int, C.c_int, _f64p]),
    ("rocp_stream_t_len", C.c_int64, [_vp]),
    ("rocp_stream_regularized", C.c_int, [_vp]),
    ("rocp_stream_last_residuals", C.c_int, [_vp, _f64p]),
    ("rocp_stream_checkpoint", C.c_int, [_vp]),
    ("rocp_stream_restore", C.c_int, [_vp]),
    ("rocp_timer_record", C.c_int, [_vp, C.c_int]),
    ("rocp_timer_elapsed_ms", C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    ("rocp_cuda_stream", _vp, [_vp]),
    ("rocp_host_alloc", _vp, [C.c_size_t]),
    ("rocp_host_free", None, [_vp, C.c_size_t]),
    ("rocp_stream_set_residual_tracking", C.c_int, [_vp, C.c_int]),
    ("rocp_stream_time_gather", C.c_int, [_vp, C.c_int]),
    ("rocp_stream_gather_times", C.c_int, [_vp, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int)]),
    ("rocp_stream_chain_times", C.c_int, [_vp, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int)]),
    ("rocp_stream_last_gather_sms", C.c_int, [_vp, C.POINTER(C.c_int)]),
    ("rocp_stream_gather_window", C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_uint32,
                                            C.c_int, C.POINTER(C.c_float)]),
    ("rocp_stream_window_bytes", C.c_int, [_vp, _i64p, _i64p]),
    ("rocp_stream_chain_trace", C.c_int, [_vp, C.c_int, C.POINTER(C.c_uint64), C.c_int64, _i64p]),
]


def build(verbose=False):
    """Compile librocp_b200.so for sm_100a (nvcc cross-compiles without a GPU)."""
    r = subprocess.run(["make", "-C", _HERE], capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError("building librocp_b200.so failed:\n" + (r.stdout or "") + (r.stderr or ""))


_lib = None


def lib():
    """Load librocp_b200.so; raise if it is missing (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2007_10798_b200); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class RocpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[rocp status {code}] {msg}")
        self.code = code


class DomainError(RocpError, ValueError):
    """std::domain_error in the reference."""


class NumericalError(RocpError):
    """rocp::NumericalError (errors.hpp:10-20); carries the sweep."""

    def __init__(self, code, msg, sweep=0):
        super().__init__(code, msg)
        self.sweep = sweep


class RecordError(RocpError, OSError):
    """File record errors (std::runtime_error in tensor_io.cpp / rocp.cpp)."""


def _check(dev_handle, rc, sweep=0):
    if rc == OK:
        return
    msg = lib().rocp_last_error(dev_handle)
    msg = msg.decode() if msg else ""
    if rc == E_DOMAIN:
        raise DomainError(rc, msg)
    if rc == E_NUMERICAL:
        raise NumericalError(rc, msg, sweep)
    if rc == E_IO:
        raise RecordError(rc, msg)
    raise RocpError(rc, msg)


def _p(a, t=_f64p):
    return a.ctypes.data_as(t)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.asfortranarray(a, dtype=np.float64)


def _ptr_array(mats):
    arr = (_f64p * max(len(mats), 1))()
    for k, m in enumerate(mats):
        arr[k] = m.ctypes.data_as(_f64p)
    return arr


def auto_sample_count(rank):
    """s = max(R, ceil(10 R ln R)) (sampling.cpp:40-45)."""
    if rank < 1:
        raise DomainError(E_DOMAIN, "rank must be positive")
    return max(rank, int(np.ceil(10.0 * rank * np.log(float(rank)))))


_live_devices = weakref.WeakSet()


@atexit.register
def _close_all_devices():
    """Deterministic teardown before interpreter finalization: streams and
    tensors are released before their handle, handles before the CUDA runtime."""
    for d in list(_live_devices):
        try:
            d.close()
        except Exception:
            pass


class Device:
    """One handle per GPU (rocp_dev)."""

    def __init__(self, device=0, world=1, rank=0, nccl_id=None, emulated=False):
        """world > 1: one handle per GPU of a mode-1 sharded job; nccl_id = rank 0's
        nccl_unique_id() bytes, broadcast by any host transport.  emulated=True: rank
        `rank` of `world` emulated on `device` (no NCCL; rocp_create_emulated_rank),
        driven with emulated_group_consume_range."""
        h = C.c_void_p()
        if emulated:
            rc = lib().rocp_create_emulated_rank(device, world, rank, C.byref(h))
        else:
            idp = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), len(nccl_id))
            rc = lib().rocp_create(device, world, rank, idp, C.byref(h))
        if rc != OK:
            raise RocpError(rc, f"rocp_create(device={device}) failed (is a GPU visible?)")
        self.h = h
        self._children = weakref.WeakSet()  # streams/tensors freed before the handle
        _live_devices.add(self)

    def _adopt(self, obj):
        self._children.add(obj)

    def close(self):
        if getattr(self, "h", None):
            lib().rocp_synchronize(self.h)
            # streams first (they reference window arenas), then tensors
            kids = list(self._children)
            for ch in kids:
                if isinstance(ch, RocpStream):
                    ch._free()
            for ch in kids:
                ch._free()
            lib().rocp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc, sweep=0):
        _check(self.h, rc, sweep)

    def synchronize(self):
        self.check(lib().rocp_synchronize(self.h))

    @property
    def kernel_launches(self):
        return int(lib().rocp_kernel_launches(self.h))

    def set_gather_sms(self, sms):
        """SMs of the overlapped window gather (rocp_set_gather_sms; < 0 = model)."""
        self.check(lib().rocp_set_gather_sms(self.h, int(sms)))

    def set_chain_sms(self, sms):
        """Blocks of this handle's persistent chain (rocp_set_chain_sms; 0 = every SM)."""
        self.check(lib().rocp_set_chain_sms(self.h, int(sms)))

    @property
    def sm_count(self):
        n = C.c_int(0)
        self.check(lib().rocp_sm_count(self.h, C.byref(n)))
        return n.value

    def tensor(self, dims, host=None):
        return DeviceTensor(self, dims, host)

    def read_tensor(self, path):
        """A reference tensor record (read_tensor_file, tensor_io.cpp:83-89) on the device."""
        h = C.c_void_p()
        self.check(lib().rocp_tensor_read_file(self.h, os.fsencode(path), C.byref(h)))
        return DeviceTensor(self, _record_dims(path), _handle=h)

    def decision_stats(self, reset=False):
        """[no-reg, reg, exact-eigenvalue, tier-2-used] solve_gram decisions since the last reset."""
        c = (C.c_uint64 * 4)()
        self.check(lib().rocp_decision_stats(self.h, c, int(bool(reset))))
        return [int(v) for v in c]

    def probe_random_reads(self, tensor, reads, seed=1):
        """Isolated 8-byte random reads per second over `tensor` (the gather's access ceiling)."""
        ms = C.c_float(0)
        self.check(lib().rocp_probe_random_reads(self.h, tensor.h, int(reads), seed, C.byref(ms)))
        return reads / (ms.value / 1000.0), float(ms.value)

    def timer_record(self, slot):
        self.check(lib().rocp_timer_record(self.h, slot))

    def timer_elapsed_ms(self, a, b):
        ms = C.c_float(0)
        self.check(lib().rocp_timer_elapsed_ms(self.h, a, b, C.byref(ms)))
        return float(ms.value)


# ---- the reference's binary records, host side (tensor_io.cpp:12-101) -----------
def _record_dims(path):
    with open(path, "rb") as f:
        head = f.read(9)
        if head[:4] != b"ROCP" or head[4] != 1:
            raise RecordError(E_IO, "bad tensor magic or version")
        order = int.from_bytes(head[5:9], "little")
        return [int.from_bytes(f.read(8), "little") for _ in range(order)]


def read_records(path):
    """Every matrix record of a file as column-major arrays (plus nothing of the tail)."""
    out = []
    with open(path, "rb") as f:
        data = f.read()
    pos = 0
    while len(data) - pos > 24 or (len(data) - pos > 8 and data[pos:pos + 4] == b"ROCP"):
        if data[pos:pos + 4] != b"ROCP":
            break
        order = int.from_bytes(data[pos + 5:pos + 9], "little")
        dims = [int.from_bytes(data[pos + 9 + 8 * k:pos + 17 + 8 * k], "little") for k in range(order)]
        pos += 9 + 8 * order
        n = int(np.prod(dims))
        vals = np.frombuffer(data, dtype="<f8", count=n, offset=pos).copy()
        pos += 8 * n
        out.append(vals.reshape(dims, order="F"))
    return out


def nccl_unique_id():
    """NCCL bootstrap id (bytes) for Device(world > 1); create on rank 0 only."""
    n = int(lib().rocp_nccl_id_size())
    buf = C.create_string_buffer(n)
    rc = lib().rocp_nccl_get_unique_id(buf)
    if rc != OK:
        raise RocpError(rc, "rocp_nccl_get_unique_id failed (NCCL unavailable?)")
    return buf.raw


def emulated_group_consume_range(streams, local_tensors, t0, batch, nb, seed, first_batch_id):
    """One window on every rank of an emulated group (rocp_emulated_group_consume_range):
    streams[g] / local_tensors[g] belong to the emulated-rank handles of one device."""
    w = len(streams)
    hs = (_vp * w)(*[s_.h for s_ in streams])
    xs = (_vp * w)(*[t.h for t in local_tensors])
    streams[0].dev.check(lib().rocp_emulated_group_consume_range(hs, w, xs, t0, batch, nb, seed, first_batch_id))


class HostBuffer:
    """Huge-page-backed, page-locked host buffer (rocp_host_alloc) viewed as a
    float64 numpy array; for host-slab streams."""

    def __init__(self, n_doubles):
        self.nbytes = int(n_doubles) * 8
        p = lib().rocp_host_alloc(self.nbytes)
        if not p:
            raise RocpError(E_OOM, "rocp_host_alloc failed")
        self.ptr = p
        self.array = np.ctypeslib.as_array((C.c_double * int(n_doubles)).from_address(p))

    def free(self):
        if getattr(self, "ptr", None):
            self.array = None
            lib().rocp_host_free(self.ptr, self.nbytes)
            self.ptr = None

    def __del__(self):
        self.free()


class DeviceTensor:
    """Device-resident DenseTensor (tensor.hpp:17-49), fp64, first index fastest."""

    def __init__(self, dev, dims, host=None, _handle=None, _parent=None):
        self.dev = dev
        self.dims = [int(x) for x in dims]
        self._parent = _parent
        if _handle is not None:
            self.h = _handle
            dev._adopt(self)
            return
        d = _i64(self.dims)
        h = C.c_void_p()
        hp = None
        if host is not None:
            host = np.ascontiguousarray(host, dtype=np.float64).ravel(order="K")
            if host.size != int(np.prod(self.dims)):
                raise DomainError(E_DOMAIN, "data length does not match product of extents")
            hp = _p(host)
        dev.check(lib().rocp_tensor_create(dev.h, _p(d, _i64p), len(d), hp, C.byref(h)))
        self.h = h
        dev._adopt(self)

    def _free(self):
        if getattr(self, "h", None):
            lib().rocp_tensor_free(self.h)
            self.h = None

    def __del__(self):
        self._free()

    @property
    def numel(self):
        return int(np.prod(self.dims))

    def slab(self, t0, length):
        h = C.c_void_p()
        self.dev.check(lib().rocp_tensor_slab(self.dev.h, self.h, t0, length, C.byref(h)))
        dims = list(self.dims)
        dims[-1] = length
        return DeviceTensor(self.dev, dims, _handle=h, _parent=self)

    def write(self, path):
        """The reference tensor record (write_tensor_file, tensor_io.cpp:77-81)."""
        self.dev.check(lib().rocp_tensor_write_file(self.dev.h, self.h, os.fsencode(path)))

    def rows(self, r0, r1):
        """Rows [r0, r1) of mode 1 as a new tensor (a rank's block of a sharded stream)."""
        h = C.c_void_p()
        self.dev.check(lib().rocp_tensor_rows(self.dev.h, self.h, r0, r1, C.byref(h)))
        dims = list(self.dims)
        dims[0] = r1 - r0
        return DeviceTensor(self.dev, dims, _handle=h)

    def download(self, out=None):
        if out is None:
            out = np.empty(self.numel, dtype=np.float64)
        if out.size != self.numel or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise DomainError(E_DOMAIN, "download target must be a contiguous float64 array of numel")
        self.dev.check(lib().rocp_tensor_download(self.dev.h, self.h, _p(out)))
        return out

    def upload(self, host):
        host = np.ascontiguousarray(host, dtype=np.float64).ravel(order="K")
        self.dev.check(lib().rocp_tensor_upload(self.dev.h, self.h, _p(host)))

    def generate(self, factors, snr_db=None, noise_seed=0):
        """gen_synthetic semantics (synthetic.cpp:8-31) with the given factors."""
        fs = [_f64(f) for f in factors]
        self.dev.check(lib().rocp_generate_synthetic(
            self.dev.h, self.h, _ptr_array(fs), fs[0].shape[1], 0 if snr_db is None else 1,
            0.0 if snr_db is None else float(snr_db), noise_seed))


# ---- primitives --------------------------------------------------------------
def draw_samples(dev, dims, mode, s, seed, batch=0, iteration=0):
    d = _i64(dims)
    rows = np.zeros(max(s, 1), dtype=np.int64)
    dec = np.zeros(max(s, 1) * (len(d) - 1), dtype=np.int64)
    dev.check(lib().rocp_draw_samples(dev.h, _p(d, _i64p), len(d), mode, s, seed, batch, iteration,
                                      _p(rows, _i64p), _p(dec, _i64p)))
    return rows[:s], dec[: s * (len(d) - 1)].reshape(s, len(d) - 1)


def decode_rows(dev, dims, mode, rows):
    d, r = _i64(dims), _i64(rows)
    dec = np.zeros(len(r) * (len(d) - 1), dtype=np.int64)
    dev.check(lib().rocp_decode_rows(dev.h, _p(d, _i64p), len(d), mode, _p(r, _i64p), len(r),
                                     _p(dec, _i64p)))
    return dec.reshape(len(r), len(d) - 1)


def sample_unfolding(dev, tensor, mode, rows):
    r = _i64(rows)
    out = np.zeros((tensor.dims[mode - 1], len(r)), order="F")
    dev.check(lib().rocp_sample_unfolding(dev.h, tensor.h, mode, _p(r, _i64p), len(r), _p(out)))
    return out


def sampled_khatri_rao(dev, decoded, factors):
    dec = _i64(decoded)
    fs = [_f64(f) for f in factors]
    R = fs[0].shape[1]
    rows = _i64([f.shape[0] for f in fs])
    z = np.zeros((dec.shape[0], R), order="F")
    dev.check(lib().rocp_sampled_khatri_rao(dev.h, _p(dec, _i64p), dec.shape[0], len(fs),
                                            _ptr_array(fs), _p(rows, _i64p), R, _p(z)))
    return z


def gram(dev, z):
    z = _f64(z)
    g = np.zeros((z.shape[1], z.shape[1]), order="F")
    dev.check(lib().rocp_gram(dev.h, _p(z), z.shape[0], z.shape[1], _p(g)))
    return g


def contract(dev, x, z):
    x, z = _f64(x), _f64(z)
    out = np.zeros((x.shape[0], z.shape[1]), order="F")
    dev.check(lib().rocp_contract(dev.h, _p(x), x.shape[0], x.shape[1], _p(z), z.shape[1], _p(out)))
    return out


def solve_gram(dev, g, rhs):
    g, rhs = _f64(g), _f64(rhs)
    if g.shape[0] != g.shape[1]:
        raise DomainError(E_DOMAIN, "solve_gram: gram matrix must be square")
    if rhs.shape[1] != g.shape[0]:
        raise DomainError(E_DOMAIN, "solve_gram: rhs column count must match gram size")
    out = np.zeros(rhs.shape, order="F")
    reg = C.c_int(0)
    dev.check(lib().rocp_solve_gram(dev.h, _p(g), _p(rhs), rhs.shape[0], g.shape[0], _p(out),
                                    C.byref(reg)))
    return out, bool(reg.value)


def solve_sampled_ls(dev, z, x):
    z, x = _f64(z), _f64(x)
    if x.shape[1] != z.shape[0]:
        raise DomainError(E_DOMAIN, "solve_sampled_ls: sample counts of z_s and x_s differ")
    out = np.zeros((x.shape[0], z.shape[1]), order="F")
    reg, und = C.c_int(0), C.c_int(0)
    dev.check(lib().rocp_solve_sampled_ls(dev.h, _p(z), _p(x), z.shape[0], x.shape[0], z.shape[1],
                                          _p(out), C.byref(reg), C.byref(und)))
    return out, bool(reg.value), bool(und.value)


def model_fitness(dev, tensor, factors):
    fs = [_f64(f) for f in factors]
    fit = C.c_double(0)
    dev.check(lib().rocp_model_fitness(dev.h, tensor.h, _ptr_array(fs), fs[0].shape[1],
                                       C.byref(fit)))
    return fit.value


# ---- cprand / stream -----------------------------------------------------------
class InitResult:
    """InitResult (cprand.hpp:19-26)."""

    def __init__(self, model, best_sampled_kr, best_fitness, iterations, regularized, fit_trace,
                 samples):
        self.model = model
        self.best_sampled_kr = best_sampled_kr
        self.best_sampled_factors = [model[n] for n in range(len(model) - 1)]
        self.best_fitness = best_fitness
        self.iterations = iterations
        self.regularized = regularized
        self.fit_trace = fit_trace
        self.samples = samples


def cprand_decompose(dev, tensor, rank, init_factors, seed, samples=0, tol=1e-4, max_iters=100):
    """cprand_decompose (cprand.cpp:12-69); init_factors = random_model(...) output."""
    N = len(tensor.dims)
    fs = [np.array(f, dtype=np.float64, order="F", copy=True) for f in init_factors]
    s = samples if samples > 0 else auto_sample_count(rank)
    kr = [np.zeros((s, rank), order="F") for _ in range(N - 1)]
    best, iters, reg, errs = C.c_double(0), C.c_int(0), C.c_int(0), C.c_int(0)
    trace = np.zeros(max(max_iters, 1))
    rc = lib().rocp_cprand(dev.h, tensor.h, rank, samples, tol, max_iters, seed, _ptr_array(fs),
                           _ptr_array(kr), C.byref(best), C.byref(iters), C.byref(reg),
                           C.byref(errs), _p(trace))
    dev.check(rc, sweep=errs.value)
    return InitResult(fs, kr, best.value, iters.value, bool(reg.value), trace[: iters.value], s)


class RocpStream:
    """RocpStream (rocp.hpp:85-107), device-resident state."""

    def __init__(self, dev, init=None, s=None, literal_init=False, t_capacity=0,
                 from_device_init=False):
        self.dev = dev
        h = C.c_void_p()
        if from_device_init:
            dev.check(lib().rocp_stream_create_from_init(dev.h, int(literal_init), t_capacity,
                                                         C.byref(h)))
            self.h = h
            dev._adopt(self)
            self.order = int(init.order) if hasattr(init, "order") else None
            self._shape_from(init)
            return
        model = init.model
        self.order = len(model)
        self.rank = model[0].shape[1]
        self.head = [m.shape[0] for m in model[:-1]]
        s = init.samples if s is None else s
        fs = [_f64(f) for f in model]
        kr = [_f64(z) for z in init.best_sampled_kr]
        for z in kr:
            if z.shape[0] != s:
                raise DomainError(E_DOMAIN, "init_state: sampled Khatri-Rao row count differs from s")
        hd = _i64(self.head)
        t_init = model[-1].shape[0]
        dev.check(lib().rocp_stream_create(dev.h, self.order, _p(hd, _i64p), self.rank, s,
                                           int(literal_init), _ptr_array(fs), t_init,
                                           _ptr_array(kr), int(init.regularized),
                                           max(t_capacity, t_init), C.byref(h)))
        self.h = h
        self.s = s
        dev._adopt(self)

    def _shape_from(self, init):
        model = init.model
        self.order = len(model)
        self.rank = model[0].shape[1]
        self.head = [m.shape[0] for m in model[:-1]]
        self.s = init.samples

    def _free(self):
        if getattr(self, "h", None):
            lib().rocp_stream_free(self.h)
            self.h = None

    def __del__(self):
        self._free()

    def shard(self, virtual_shards=8):
        """Mode-1 sharding across Device(world, rank) (rocp_stream_shard): this rank
        keeps U(1)/P(1) rows [row0, row1); consume takes the rank's local tensor."""
        self.dev.check(lib().rocp_stream_shard(self.h, virtual_shards))
        v, r0, r1 = C.c_int(0), C.c_int64(0), C.c_int64(0)
        self.dev.check(lib().rocp_stream_shard_info(self.h, C.byref(v), C.byref(r0), C.byref(r1)))
        self.virtual_shards, self.row0, self.row1 = v.value, r0.value, r1.value
        self.head = [self.row1 - self.row0] + list(self.head[1:])
        return self.row0, self.row1

    def _check_mode(self, mode):
        if not 1 <= mode < self.order:
            raise DomainError(E_DOMAIN, "update_mode_with: index set must be over a non-temporal mode")

    def consume(self, x_new, seed, batch_id):
        if isinstance(x_new, DeviceTensor):
            self.dev.check(lib().rocp_stream_consume(self.h, x_new.h, seed, batch_id))
        else:
            x = np.ascontiguousarray(x_new, dtype=np.float64).ravel(order="K")
            head = int(np.prod(self.head))
            if x.size % head:
                raise DomainError(E_DOMAIN, "batch head extents do not match stream")
            self.dev.check(lib().rocp_stream_consume_host(self.h, _p(x), x.size // head, seed,
                                                          batch_id))

    def consume_range(self, x, t0, batch, nb, seed, first_batch_id):
        self.dev.check(lib().rocp_stream_consume_range(self.h, x.h, t0, batch, nb, seed,
                                                       first_batch_id))

    def consume_range_host(self, x, batch, nb, seed, first_batch_id, threads=0):
        """nb consecutive host slabs of `batch` slices (flat, first index fastest)."""
        x = np.ascontiguousarray(x, dtype=np.float64).ravel(order="K")
        if x.size != int(np.prod(self.head)) * batch * nb:
            raise DomainError(E_DOMAIN, "host range size does not match head dims x batch x nb")
        self.dev.check(lib().rocp_stream_consume_range_host(self.h, _p(x), batch, nb, seed, first_batch_id,
                                                            threads))

    def update_last_mode_with(self, x_new, rows):
        r = _i64(rows)
        B = x_new.dims[-1]
        u = np.zeros((B, self.rank), order="F")
        z = np.zeros((len(r), self.rank), order="F")
        reg = C.c_int(0)
        self.dev.check(lib().rocp_stream_update_last_mode_with(self.h, x_new.h, _p(r, _i64p), len(r),
                                                               _p(u), _p(z), C.byref(reg)))
        return u, z, bool(reg.value)

    def append_temporal(self, u_new):
        u = _f64(u_new)
        self.dev.check(lib().rocp_stream_append_temporal(self.h, _p(u), u.shape[0]))

    def update_mode_with(self, x_new, u_new, mode, rows):
        self._check_mode(mode)
        r = _i64(rows)
        u = _f64(u_new)
        z = np.zeros((len(r), self.rank), order="F")
        xs = np.zeros((self.head[mode - 1], len(r)), order="F")
        reg = C.c_int(0)
        self.dev.check(lib().rocp_stream_update_mode_with(self.h, x_new.h, _p(u), mode, _p(r, _i64p),
                                                          len(r), _p(z), _p(xs), C.byref(reg)))
        return z, xs, bool(reg.value)

    def finish_batch(self, batch):
        self.dev.check(lib().rocp_stream_finish_batch(self.h, batch))

    def _get(self, what, mode, shape):
        out = np.zeros(shape, order="F")
        self.dev.check(lib().rocp_stream_get(self.h, what, mode, _p(out)))
        return out

    def factor(self, mode):
        return self._get(0, mode, (self.head[mode - 1], self.rank))

    def p(self, mode):
        return self._get(1, mode, (self.head[mode - 1], self.rank))

    def q(self, mode):
        return self._get(2, mode, (self.rank, self.rank))

    def temporal(self):
        return self._get(3, 0, (self.t_len, self.rank))

    def set(self, what, mode, arr):
        a = _f64(arr)
        self.dev.check(lib().rocp_stream_set(self.h, what, mode, _p(a)))

    def model(self):
        """RocpStream::model (rocp.cpp:162-168)."""
        return [self.factor(n) for n in range(1, self.order)] + [self.temporal()]

    @property
    def t_len(self):
        return int(lib().rocp_stream_t_len(self.h))

    @property
    def regularized(self):
        return bool(lib().rocp_stream_regularized(self.h))

    def last_residuals(self):
        out = np.zeros(self.order)
        self.dev.check(lib().rocp_stream_last_residuals(self.h, _p(out)))
        return out

    def set_residual_tracking(self, enable):
        self.dev.check(lib().rocp_stream_set_residual_tracking(self.h, int(enable)))

    def time_gather(self, enable):
        self.dev.check(lib().rocp_stream_time_gather(self.h, int(enable)))

    def gather_times(self, max_n=4096):
        buf = (C.c_float * max_n)()
        cnt = C.c_int(0)
        self.dev.check(lib().rocp_stream_gather_times(self.h, buf, max_n, C.byref(cnt)))
        return [float(buf[k]) for k in range(min(cnt.value, max_n))]

    @property
    def last_gather_sms(self):
        v = C.c_int(0)
        self.dev.check(lib().rocp_stream_last_gather_sms(self.h, C.byref(v)))
        return int(v.value)

    def gather_window(self, x, t0, batch, nb, seed, first_batch_id, sms=0):
        """Profiling aid: the window gather of consume_range(...) alone on `sms` SMs
        (0 = all), event-timed; returns milliseconds (rocp_stream_gather_window)."""
        ms = C.c_float(0)
        self.dev.check(lib().rocp_stream_gather_window(self.h, x.h, t0, batch, nb, seed, first_batch_id, int(sms),
                                                       C.byref(ms)))
        return float(ms.value)

    def chain_times(self, max_n=4096):
        buf = (C.c_float * max_n)()
        cnt = C.c_int(0)
        self.dev.check(lib().rocp_stream_chain_times(self.h, buf, max_n, C.byref(cnt)))
        return [float(buf[k]) for k in range(min(cnt.value, max_n))]

    def chain_trace(self, enable=None, fetch=True):
        if enable is not None and not fetch:
            self.dev.check(lib().rocp_stream_chain_trace(self.h, int(enable), None, 0, None))
            return None
        n = C.c_int64(0)
        self.dev.check(lib().rocp_stream_chain_trace(self.h, int(bool(enable)), None, 0, C.byref(n)))
        buf = np.zeros(max(n.value, 1), dtype=np.uint64)
        self.dev.check(lib().rocp_stream_chain_trace(self.h, int(bool(enable)),
                                                     buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                     n.value, C.byref(n)))
        return buf[: n.value].reshape(-1, 24)  # kTraceSlots stamps per (batch, stage)

    def window_bytes(self):
        u, e = C.c_int64(0), C.c_int64(0)
        self.dev.check(lib().rocp_stream_window_bytes(self.h, C.byref(u), C.byref(e)))
        return int(u.value), int(e.value)

    def write_state(self, path):
        """save_state record of the ComplementaryState (rocp.cpp:180-184)."""
        self.dev.check(lib().rocp_stream_write_state(self.h, os.fsencode(path)))

    def read_state(self, path):
        """load_state record (rocp.cpp:186-211) into this stream: P, Q, t_len."""
        self.dev.check(lib().rocp_stream_read_state(self.h, os.fsencode(path)))

    def consume_file(self, path, t0, batch, nb, seed, first_batch_id, threads=0):
        """nb batches of `batch` slices from a tensor record file, starting at slice t0."""
        self.dev.check(lib().rocp_stream_consume_file(self.h, os.fsencode(path), t0, batch, nb, seed,
                                                      first_batch_id, threads))

    def write_checkpoint(self, path):
        self.dev.check(lib().rocp_stream_write_checkpoint(self.h, os.fsencode(path)))

    @classmethod
    def from_checkpoint(cls, dev, path, t_capacity=0):
        """A stream resumed from write_checkpoint's record."""
        h = C.c_void_p()
        dev.check(lib().rocp_stream_create_from_checkpoint(dev.h, os.fsencode(path), t_capacity, C.byref(h)))
        st = cls.__new__(cls)
        st.dev, st.h = dev, h
        dev._adopt(st)
        recs = read_records(path)
        N = (len(recs) - 1) // 3 + 1
        st.order = N
        st.rank = recs[0].shape[1]
        st.head = [recs[n].shape[0] for n in range(N - 1)]
        st.s = None
        return st

    def checkpoint(self):
        self.dev.check(lib().rocp_stream_checkpoint(self.h))

    def restore(self):
        self.dev.check(lib().rocp_stream_restore(self.h))
