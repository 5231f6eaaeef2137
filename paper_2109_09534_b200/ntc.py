"""Python mirror of the reference's proj/core API for the hot path, running on
the B200 through the C-ABI (libntcb.so).  Names, argument meaning and error
behaviour follow the reference so that tests read like its own:

  reference (C++)                           here
  ntc::RngStream          rng.hpp:13-63      RngStream (host stream-state helper)
  ntc::sweep_stream       ao.cpp:65-68       sweep_stream
  ntc::NmcConfig          nmc.hpp:13-23      NmcConfig
  ntc::AoConfig           ao.hpp:12-29       AoConfig
  ntc::MetricsRecord      ao.hpp:31-37       MetricsRecord
  ntc::SparseTensor       sparse_tensor.hpp  SparseTensor   (validated/sorted on device)
  ntc::ModeView           mode_view.hpp      SparseTensor.view(mode) (device-built)
  ntc::FactorSet          factor_set.hpp     FactorSet
  ntc::initial_factors    ao.cpp:70-73       initial_factors
  ntc::sample_row         nmc.hpp:45         sample_row
  ntc::s_nmc              nmc.hpp:93-95      s_nmc
  ntc::ao_ntc             ao.hpp:67-68       ao_ntc
  ntc::objective          metrics.hpp:9      objective
  ntc::relative_error     metrics.hpp:13     relative_error
  ntc::epoch_fraction / term_cond            epoch_fraction / term_cond

Exceptions: std::invalid_argument -> InvalidArgument (ValueError),
std::runtime_error -> NtcRuntimeError, std::out_of_range -> OutOfRange
(IndexError), std::domain_error -> DomainError (ArithmeticError).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from ._lib import (AoConfigC, DomainError, InvalidArgument, MetricsRecordC, NmcConfigC,
                   NtcRuntimeError, OutOfRange, check, f32p, f64p, u32p, u64p)

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class RngStream:
    """Host-side splitmix64 stream identical to ntc::RngStream; only used to
    derive the raw 64-bit states that cross the C-ABI (plus the reference's
    ``state`` accessor that rng.hpp lacks)."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def fork(self, tag: int) -> "RngStream":
        return RngStream(_mix(self.state ^ ((GOLDEN * (tag + 1)) & M64)))

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & M64
        return _mix(self.state)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def sweep_stream(seed: int, sweep: int, mode: int) -> RngStream:
    return RngStream(seed).fork(2).fork(sweep).fork(mode)


@dataclass
class NmcConfig:
    lambda_: float = 1e-3
    c: float = 1.0
    max_inner: int = 1
    power_iters: int = 30
    power_tol: float = 1e-6
    threads: int = 1
    chunk: int = 0

    def validate(self) -> None:  # nmc.cpp:13-23
        if not (self.lambda_ > 0.0):
            raise InvalidArgument("NmcConfig: lambda must be > 0")
        if not (0.0 < self.c <= 1.0):
            raise InvalidArgument("NmcConfig: c must be in (0, 1]")
        if self.max_inner < 0:
            raise InvalidArgument("NmcConfig: max_inner must be >= 0")
        if self.power_iters < 1:
            raise InvalidArgument("NmcConfig: power_iters must be >= 1")
        if not (self.power_tol > 0.0):
            raise InvalidArgument("NmcConfig: power_tol must be > 0")
        if self.threads < 1:
            raise InvalidArgument("NmcConfig: threads must be >= 1")
        if self.chunk < 0:
            raise InvalidArgument("NmcConfig: chunk must be >= 0")

    def c_struct(self) -> NmcConfigC:
        return NmcConfigC(self.lambda_, self.c, self.max_inner, self.power_iters, self.power_tol,
                          self.threads, self.chunk)


@dataclass
class AoConfig:
    rank: int = 1
    lambda_: float = 1e-3
    c: float = 1.0
    max_inner: int = 1
    max_epochs: float = 100.0
    term_tol: float = 0.0
    seed: int = 0
    threads: int = 1
    chunk: int = 0
    power_iters: int = 30
    power_tol: float = 1e-6
    eval_metrics: bool = True
    metrics_every: int = 1

    def nmc(self) -> NmcConfig:  # ao.cpp:40-50
        return NmcConfig(self.lambda_, self.c, self.max_inner, self.power_iters, self.power_tol,
                         self.threads, self.chunk)

    def validate(self) -> None:  # ao.cpp:30-38
        if self.rank == 0:
            raise InvalidArgument("AoConfig: rank must be positive")
        if not (self.max_epochs >= 0.0):
            raise InvalidArgument("AoConfig: max_epochs must be >= 0")
        if not (self.term_tol >= 0.0):
            raise InvalidArgument("AoConfig: term_tol must be >= 0")
        if self.metrics_every < 1:
            raise InvalidArgument("AoConfig: metrics_every must be >= 1")
        self.nmc().validate()

    def c_struct(self) -> AoConfigC:
        return AoConfigC(self.rank, self.lambda_, self.c, self.max_inner, self.power_iters,
                         self.max_epochs, self.term_tol, self.seed, self.threads, self.chunk,
                         self.power_tol, int(self.eval_metrics), self.metrics_every)


@dataclass
class MetricsRecord:
    epoch: float = 0.0
    objective: float = math.nan
    rel_error: float = math.nan
    wall_seconds: float = 0.0
    entries_accessed: int = 0


@dataclass
class SnmcStats:
    entries_accessed: int = 0


def epoch_fraction(entries_accessed: int, omega_size: int) -> float:  # ao.cpp:52-56
    if omega_size == 0:
        raise InvalidArgument("epoch_fraction: empty observation set")
    return entries_accessed / omega_size


def _plateau(h: List[MetricsRecord], tol: float) -> bool:  # ao.cpp:21-26
    if len(h) < 4:
        return False
    for t in range(len(h) - 3, len(h)):
        if not (abs(h[t].rel_error - h[t - 1].rel_error) < tol):
            return False
    return True


def term_cond(history: List[MetricsRecord], cfg: AoConfig) -> bool:  # ao.cpp:58-63
    if not history:
        raise InvalidArgument("term_cond: needs at least one record")
    if history[-1].epoch >= cfg.max_epochs:
        return True
    return _plateau(history, cfg.term_tol)


# --------------------------------------------------------------------------
class PinnedArray(np.ndarray):
    """numpy array over page-locked host memory (ntcb_host_alloc), freed with
    the array; host-buffer S_NMC calls on such arrays take the device-side
    conversion path (no host staging)."""

    def __new__(cls, shape, dtype=np.float64):
        L = _lib.load()
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        p = C.c_void_p()
        check(L.ntcb_host_alloc(n, C.byref(p)))
        buf = (C.c_char * max(n, 1)).from_address(p.value)
        obj = np.ndarray.__new__(cls, shape, dt, buffer=buf)
        obj._ptr = p.value
        obj._owner = True
        return obj

    def __array_finalize__(self, obj):
        self._ptr = getattr(obj, "_ptr", None)
        self._owner = False  # views never free

    def __del__(self):
        if getattr(self, "_owner", False) and self._ptr:
            try:
                _lib.load().ntcb_host_free(C.c_void_p(self._ptr))
            except Exception:
                pass
            self._ptr = None


def pinned_like(a) -> "PinnedArray":
    out = PinnedArray(np.shape(a), np.asarray(a).dtype)
    out[...] = a
    return out


class Context:
    """An ntcb_context: one device, one stream, a resident tensor + factors."""

    def __init__(self, device: int = 0):
        self.L = _lib.load()
        h = C.c_void_p()
        check(self.L.ntcb_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.ntcb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # launch policy (ntcb_tuning; never changes results) ------------------
    def tuning(self) -> dict:
        t = _lib.TuningC()
        check(self.L.ntcb_get_tuning(self.h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in _lib.TuningC._fields_}

    def set_tuning(self, **kw) -> None:
        """Change launch-policy knobs (A/B measurements), e.g.
        set_tuning(no_tc=1) or set_tuning(heavy_win_log2=16)."""
        t = _lib.TuningC()
        check(self.L.ntcb_get_tuning(self.h, C.byref(t)))
        for k, v in kw.items():
            if k not in dict(_lib.TuningC._fields_):
                raise InvalidArgument(f"tuning: unknown field {k}")
            setattr(t, k, int(v))
        check(self.L.ntcb_set_tuning(self.h, C.byref(t)))

    # tensor -------------------------------------------------------------
    def load(self, dims, indices, values):
        dims = np.ascontiguousarray(dims, np.uint64)
        idx = np.ascontiguousarray(indices, np.uint32).reshape(-1)
        nnz = 0 if len(dims) == 0 else (idx.size // max(len(dims), 1))
        if np.asarray(values).dtype == np.float32:
            vals = np.ascontiguousarray(values, np.float32)
            check(self.L.ntcb_tensor_load_f32(self.h, len(dims), dims.ctypes.data_as(u64p),
                                              len(vals), idx.ctypes.data_as(u32p),
                                              vals.ctypes.data_as(f32p)))
        else:
            vals = np.ascontiguousarray(values, np.float64)
            if idx.size != vals.size * len(dims):
                raise InvalidArgument("SparseTensor: index/value length mismatch")
            check(self.L.ntcb_tensor_load(self.h, len(dims), dims.ctypes.data_as(u64p), len(vals),
                                          idx.ctypes.data_as(u32p), vals.ctypes.data_as(f64p)))
        del nnz

    def synth_uniform(self, dims, nnz, true_rank, sigma, seed):
        dims = np.ascontiguousarray(dims, np.uint64)
        check(self.L.ntcb_synth_uniform(self.h, len(dims), dims.ctypes.data_as(u64p), nnz,
                                        true_rank, sigma, seed))

    def synth(self, dims, nnz, true_rank, sigma, seed, zipf_alpha=None, value_kind=0):
        dims = np.ascontiguousarray(dims, np.uint64)
        za = None
        if zipf_alpha is not None:
            za = np.ascontiguousarray(zipf_alpha, np.float64)
        check(self.L.ntcb_synth(self.h, len(dims), dims.ctypes.data_as(u64p), nnz, true_rank,
                                sigma, seed, None if za is None else za.ctypes.data_as(f64p),
                                value_kind))

    def info(self):
        order = C.c_int()
        dims = np.zeros(8, np.uint64)
        nnz = C.c_uint64()
        check(self.L.ntcb_tensor_info(self.h, C.byref(order), dims.ctypes.data_as(u64p),
                                      C.byref(nnz)))
        return order.value, [int(d) for d in dims[: order.value]], nnz.value

    def view(self, mode):
        order, dims, nnz = self.info()
        off = np.zeros(dims[mode] + 1, np.uint64)
        oth = np.zeros(max(nnz * (order - 1), 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float32)
        check(self.L.ntcb_view_export(self.h, mode, off.ctypes.data_as(u64p),
                                      oth.ctypes.data_as(u32p), val.ctypes.data_as(f32p)))
        return off, oth[: nnz * (order - 1)].reshape(nnz, order - 1), val[:nnz]

    def view_offsets(self, mode):
        order, dims, nnz = self.info()
        off = np.zeros(dims[mode] + 1, np.uint64)
        check(self.L.ntcb_view_export(self.h, mode, off.ctypes.data_as(u64p), None, None))
        return off

    def view_rows(self, mode, row_begin, row_end):
        """(offsets rebased to 0, others, values) of the slices of rows [row_begin, row_end)."""
        order, dims, nnz = self.info()
        off = np.zeros(row_end - row_begin + 1, np.uint64)
        check(self.L.ntcb_view_export_rows(self.h, mode, row_begin, row_end,
                                           off.ctypes.data_as(u64p), None, None))
        n = int(off[-1] - off[0])
        oth = np.zeros(max(n * (order - 1), 1), np.uint32)
        val = np.zeros(max(n, 1), np.float32)
        check(self.L.ntcb_view_export_rows(self.h, mode, row_begin, row_end, None,
                                           oth.ctypes.data_as(u32p), val.ctypes.data_as(f32p)))
        return off - off[0], oth[: n * (order - 1)].reshape(n, order - 1), val[:n]

    def view_keep_rows(self, mode, row_begin, row_end):
        """Slab storage (ntcb_view_keep_rows): only rows [row_begin, row_end)
        of view `mode` stay on the device."""
        check(self.L.ntcb_view_keep_rows(self.h, mode, row_begin, row_end))

    def view_resident(self, mode):
        """(row_begin, row_end, device bytes) of the resident part of a view."""
        a, b, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(self.L.ntcb_view_resident(self.h, mode, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def set_stream(self, stream_ptr):
        check(self.L.ntcb_set_stream(self.h, C.c_void_p(stream_ptr)))

    def canonical(self):
        order, dims, nnz = self.info()
        idx = np.zeros(max(nnz * order, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float32)
        check(self.L.ntcb_tensor_export(self.h, idx.ctypes.data_as(u32p), val.ctypes.data_as(f32p)))
        return idx[: nnz * order].reshape(nnz, order), val[:nnz]

    # factors ------------------------------------------------------------
    def set_factors(self, rank, factors, momentum=None):
        fs = [np.ascontiguousarray(f, np.float64) for f in factors]
        ptrs = (f64p * len(fs))(*[f.ctypes.data_as(f64p) for f in fs])
        mptrs = None
        if momentum is not None:
            ms = [np.ascontiguousarray(f, np.float64) for f in momentum]
            mptrs = (f64p * len(ms))(*[f.ctypes.data_as(f64p) for f in ms])
        check(self.L.ntcb_factors_init(self.h, rank, ptrs, mptrs))
        self.rank = rank

    def random_factors(self, rank, seed):
        check(self.L.ntcb_factors_random(self.h, rank, seed))
        self.rank = rank

    def set_factor(self, mode, a=None, y=None):
        a = None if a is None else np.ascontiguousarray(a, np.float64)
        y = None if y is None else np.ascontiguousarray(y, np.float64)
        check(self.L.ntcb_factor_set(self.h, mode, None if a is None else a.ctypes.data_as(f64p),
                                     None if y is None else y.ctypes.data_as(f64p)))

    def get_factor(self, mode):
        order, dims, _ = self.info()
        a = np.zeros((dims[mode], self.rank), np.float64)
        y = np.zeros((dims[mode], self.rank), np.float64)
        check(self.L.ntcb_factor_get(self.h, mode, a.ctypes.data_as(f64p), y.ctypes.data_as(f64p)))
        return a, y

    def factor_device_ptr(self, mode, which=0):
        p = C.c_void_p()
        ld = C.c_uint64()
        check(self.L.ntcb_factor_device_ptr(self.h, mode, which, C.byref(p), C.byref(ld)))
        return p.value, ld.value

    # fused exchange (row-sharded multi-GPU) ------------------------------
    def factor_ipc_handle(self, mode) -> bytes:
        buf = (C.c_ubyte * 64)()
        check(self.L.ntcb_factor_ipc_handle(self.h, mode, buf))
        return bytes(buf)

    def ipc_open(self, handle: bytes) -> int:
        buf = (C.c_ubyte * 64).from_buffer_copy(handle)
        p = C.c_void_p()
        check(self.L.ntcb_ipc_open(self.h, buf, C.byref(p)))
        return p.value

    def set_factor_peers(self, mode, ptrs):
        arr = (C.c_void_p * max(len(ptrs), 1))(*ptrs)
        check(self.L.ntcb_factor_set_peers(self.h, mode, len(ptrs), arr))

    # solver -------------------------------------------------------------
    def s_nmc(self, mode, cfg: NmcConfig, rng_state: int, a_init=None) -> int:
        acc = C.c_uint64(0)
        cs = cfg.c_struct()
        ai = None
        if a_init is not None:
            ai = np.ascontiguousarray(a_init, np.float64)
        check(self.L.ntcb_s_nmc(self.h, mode, None if ai is None else ai.ctypes.data_as(f64p),
                                C.byref(cs), rng_state, C.byref(acc)))
        return acc.value

    def s_nmc_host(self, mode, a_init, a_out, y_out, cfg: NmcConfig, rng_state: int) -> int:
        """Host-buffer drop-in (ntcb_s_nmc_host): float64 (rows, R) arrays in/out."""
        acc = C.c_uint64(0)
        cs = cfg.c_struct()
        check(self.L.ntcb_s_nmc_host(self.h, mode, a_init.ctypes.data_as(f64p),
                                     a_out.ctypes.data_as(f64p), y_out.ctypes.data_as(f64p),
                                     C.byref(cs), rng_state, C.byref(acc)))
        return acc.value

    def sample_prefetch(self, mode, cfg: NmcConfig, rng_state: int) -> None:
        """Hint (ntcb_sample_prefetch): draw the first sampled set of a future
        s_nmc / s_nmc_host call (same mode, c, rng_state) now, on the sampler
        stream.  Results are unchanged."""
        cs = cfg.c_struct()
        check(self.L.ntcb_sample_prefetch(self.h, mode, C.byref(cs), rng_state))

    def s_nmc_rows_async(self, mode, row_begin, row_end, cfg: NmcConfig, rng_state: int):
        cs = cfg.c_struct()
        check(self.L.ntcb_s_nmc_rows_async(self.h, mode, row_begin, row_end, C.byref(cs), rng_state))

    def segment_length(self, mode) -> int:
        v = C.c_uint64()
        check(self.L.ntcb_segment_length(self.h, mode, C.byref(v)))
        return v.value

    def s_nmc_chunks_async(self, mode, row, chunk_begin, chunk_end, cfg: NmcConfig, rng_state: int, d_slots: int):
        """Chunks [chunk_begin, chunk_end) of a shared heavy row: fp32 (H, w)
        partials ((R*R + R) floats per chunk) into the device buffer d_slots."""
        cs = cfg.c_struct()
        check(self.L.ntcb_s_nmc_chunks_async(self.h, mode, row, chunk_begin, chunk_end, C.byref(cs), rng_state,
                                             C.c_void_p(d_slots)))

    def finalize_row_async(self, mode, row, d_slots: int, nslots, cfg: NmcConfig):
        cs = cfg.c_struct()
        check(self.L.ntcb_finalize_row_async(self.h, mode, row, C.c_void_p(d_slots), nslots, C.byref(cs)))

    def sweep_async(self, sweep, cfg: NmcConfig, seed):
        cs = cfg.c_struct()
        check(self.L.ntcb_sweep_async(self.h, sweep, C.byref(cs), seed))

    def collect(self) -> int:
        acc = C.c_uint64(0)
        check(self.L.ntcb_collect(self.h, C.byref(acc)))
        return acc.value

    def sample_rows(self, mode, c, rng_state, l=0, row_begin=0, row_end=None):
        order, dims, _ = self.info()
        row_end = dims[mode] if row_end is None else row_end
        po = np.zeros(row_end - row_begin + 1, np.uint64)
        check(self.L.ntcb_sample_rows(self.h, mode, c, rng_state, l, row_begin, row_end,
                                      po.ctypes.data_as(u64p), None))
        picks = np.zeros(max(int(po[-1]), 1), np.uint32)
        check(self.L.ntcb_sample_rows(self.h, mode, c, rng_state, l, row_begin, row_end,
                                      po.ctypes.data_as(u64p), picks.ctypes.data_as(u32p)))
        return po, picks[: int(po[-1])]

    def sample_mask(self, mode, c, rng_state, l=0, row_begin=0, row_end=None):
        """Production sampled-set mask for rows [row_begin, row_end): returns
        (first entry position e0, boolean array over entries [e0, e1))."""
        off = self.view_offsets(mode)
        row_end = len(off) - 1 if row_end is None else row_end
        e0, e1 = int(off[row_begin]), int(off[row_end])
        if e1 <= e0:
            return e0, np.zeros(0, bool)
        w0, w1 = e0 >> 5, ((e1 - 1) >> 5) + 1
        words = np.zeros(w1 - w0, np.uint32)
        check(self.L.ntcb_sample_mask(self.h, mode, c, rng_state, l, row_begin, row_end,
                                      words.ctypes.data_as(u32p)))
        bits = np.unpackbits(words.view(np.uint8), bitorder="little").astype(bool)
        return e0, bits[e0 - 32 * w0: e1 - 32 * w0]

    def sample_row(self, mode, row, c, row_state):
        cnt = C.c_uint64()
        check(self.L.ntcb_sample_row(self.h, mode, row, c, row_state, None, C.byref(cnt)))
        picks = np.zeros(max(cnt.value, 1), np.uint32)
        check(self.L.ntcb_sample_row(self.h, mode, row, c, row_state, picks.ctypes.data_as(u32p),
                                     C.byref(cnt)))
        return picks[: cnt.value]

    def metrics(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(self.L.ntcb_metrics(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def objective(self, lam):
        out = C.c_double()
        check(self.L.ntcb_objective(self.h, lam, C.byref(out)))
        return out.value

    def relative_error(self):
        out = C.c_double()
        check(self.L.ntcb_relative_error(self.h, C.byref(out)))
        return out.value

    def rmse(self):
        out = C.c_double()
        check(self.L.ntcb_rmse(self.h, C.byref(out)))
        return out.value

    def ao_ntc(self, cfg: AoConfig, observer=None, max_history=1 << 16):
        hist = (MetricsRecordC * max_history)()
        n = C.c_uint64()
        cs = cfg.c_struct()

        def _obs(rec, ctx, user):
            r = rec.contents
            observer(MetricsRecord(r.epoch, r.objective, r.rel_error, r.wall_seconds,
                                   r.entries_accessed))

        cb = _lib.OBSERVER(_obs) if observer else _lib.OBSERVER()
        check(self.L.ntcb_ao_ntc(self.h, C.byref(cs), hist, max_history, C.byref(n), cb, None))
        return [MetricsRecord(h.epoch, h.objective, h.rel_error, h.wall_seconds, h.entries_accessed)
                for h in hist[: min(n.value, max_history)]]

    def render_model(self) -> np.ndarray:
        """render_model (image.cpp:161-183): (H, W, 3) uint8 pixels of the
        resident factors of an H x W x 3 tensor."""
        order, dims, _ = self.info()
        H, W = (dims[0], dims[1]) if order >= 2 else (0, 0)
        out = np.zeros(max(3 * H * W, 1), np.uint8)
        check(self.L.ntcb_render_model(self.h, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out[: 3 * H * W].reshape(H, W, 3)

    def profile(self, on=True):
        check(self.L.ntcb_profile_enable(self.h, int(on)))

    def profile_read_kernel(self):
        """(ms, launches) of the update's item kernel alone since profiling was enabled."""
        t, n = C.c_double(), C.c_uint64()
        check(self.L.ntcb_profile_read_kernel(self.h, C.byref(t), C.byref(n)))
        return t.value, n.value

    def profile_read(self):
        u, s = C.c_double(), C.c_double()
        n, nu = C.c_uint64(), C.c_uint64()
        check(self.L.ntcb_profile_read(self.h, C.byref(u), C.byref(s), C.byref(n), C.byref(nu)))
        return u.value, s.value, n.value, nu.value


# --------------------------------------------------------------------------
# Reference-shaped objects
# --------------------------------------------------------------------------
class SparseTensor:
    """ntc::SparseTensor: validated, lexicographically sorted COO, with the
    mode views built on the device at construction (sparse_tensor.cpp:24-73,
    mode_view.cpp:8-37).  Coordinates 0-based, values stored in fp32."""

    def __init__(self, dims, indices, values, device: int = 0):
        dims = [int(d) for d in dims]
        idx = np.asarray(indices, np.uint32).reshape(-1)
        vals = np.asarray(values)
        if len(dims) >= 2 and idx.size != vals.size * len(dims):
            raise InvalidArgument("SparseTensor: index/value length mismatch")
        self.ctx = Context(device)
        self.ctx.load(dims, idx, vals)
        self._dims = dims

    def order(self):
        return len(self._dims)

    def dims(self):
        return list(self._dims)

    def nnz(self):
        return self.ctx.info()[2]

    def indices(self):
        return self.ctx.canonical()[0]

    def values(self):
        return self.ctx.canonical()[1]

    def view(self, mode):
        return self.ctx.view(mode)

    def observed_norm(self):
        v = self.values().astype(np.float64)
        return float(np.sqrt(np.sum(v * v)))


def parse_tns(path: str):
    """Parallel host parse of a .tns file (ntcb_tns_parse; read_tns syntax and
    diagnostics, tns_io.cpp:41-125): returns (dims, indices (nnz, N) 0-based,
    values float64) in file order."""
    L = _lib.load()
    order = C.c_int()
    dims = np.zeros(8, np.uint64)
    nnz = C.c_uint64()
    ip, vp = u32p(), f64p()
    rc = L.ntcb_tns_parse(path.encode(), C.byref(order), dims.ctypes.data_as(u64p), C.byref(nnz),
                          C.byref(ip), C.byref(vp))
    if rc:
        raise _lib._EXC.get(rc, NtcRuntimeError)(L.ntcb_tns_last_error().decode())
    try:
        N, n = order.value, nnz.value
        idx = np.ctypeslib.as_array(ip, shape=(max(n * N, 1),))[: n * N].reshape(n, N).copy()
        vals = np.ctypeslib.as_array(vp, shape=(max(n, 1),))[:n].copy()
    finally:
        L.ntcb_free(C.cast(ip, C.c_void_p))
        L.ntcb_free(C.cast(vp, C.c_void_p))
    return [int(d) for d in dims[:N]], idx, vals


def read_tns(path: str, device: int = 0) -> "SparseTensor":
    """ntc::read_tns (tns_io.cpp:41-125): parse in parallel, then build the
    canonical tensor and mode views on the device."""
    dims, idx, vals = parse_tns(path)
    return SparseTensor(dims, idx, vals, device)


def write_tns(t: "SparseTensor", path: str) -> None:
    """ntc::write_tns (tns_io.cpp:127-142)."""
    L = _lib.load()
    idx, vals = t.ctx.canonical()
    dims = np.ascontiguousarray(t.dims(), np.uint64)
    idx = np.ascontiguousarray(idx, np.uint32)
    v64 = np.ascontiguousarray(vals, np.float64)
    check(L.ntcb_tns_write(path.encode(), len(dims), dims.ctypes.data_as(u64p), len(v64),
                           idx.ctypes.data_as(u32p), v64.ctypes.data_as(f64p)))


@dataclass
class FactorSet:
    rank: int = 0
    factors: List[np.ndarray] = field(default_factory=list)
    momentum: List[np.ndarray] = field(default_factory=list)

    @staticmethod
    def zeros(dims, rank) -> "FactorSet":
        if rank == 0:
            raise InvalidArgument("FactorSet: rank must be positive")
        return FactorSet(rank, [np.zeros((d, rank)) for d in dims], [np.zeros((d, rank)) for d in dims])

    @staticmethod
    def random_uniform(dims, rank, base: RngStream) -> "FactorSet":  # factor_set.cpp:18-27
        f = FactorSet.zeros(dims, rank)
        for m, d in enumerate(dims):
            s = base.fork(m)
            n = d * rank
            ctr = (s.state + GOLDEN * np.arange(1, n + 1, dtype=np.uint64)).astype(np.uint64)
            z = ctr
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            f.factors[m] = ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53).reshape(d, rank)
            f.momentum[m] = f.factors[m].copy()
        return f

    def order(self):
        return len(self.factors)

    def all_nonnegative(self):
        return all(bool(np.all(u >= 0)) for u in self.factors)

    def copy(self):
        return FactorSet(self.rank, [u.copy() for u in self.factors], [u.copy() for u in self.momentum])


def initial_factors(dims, rank, seed) -> FactorSet:  # ao.cpp:70-73
    with np.errstate(over="ignore"):
        return FactorSet.random_uniform(list(dims), rank, RngStream(seed).fork(1))


def _push_factors(t: SparseTensor, f: FactorSet):
    if f.rank == 0:
        raise InvalidArgument("FactorSet: rank must be positive")
    t.ctx.set_factors(f.rank, f.factors, f.momentum)


def sample_row(t: SparseTensor, mode: int, row: int, c: float, rng: RngStream) -> np.ndarray:
    """ntc::sample_row (nmc.cpp:110-118) on the device: the picks of one slice
    (slice-local offsets, in draw order) for the stream `rng` used as is."""
    return t.ctx.sample_row(mode, row, c, rng.state)


def s_nmc(t: SparseTensor, factors: FactorSet, mode: int, a_init, cfg: NmcConfig,
          rng: RngStream, stats: Optional[SnmcStats] = None) -> np.ndarray:
    """ntc::s_nmc (nmc.cpp:199-272) on the device; updates factors.factors[mode]
    and factors.momentum[mode] in place and returns factors.factors[mode]."""
    cfg.validate()
    if mode < 0 or mode >= factors.order():
        raise InvalidArgument("s_nmc: mode out of range")
    dims = t.dims()
    a_init = np.asarray(a_init, np.float64)
    if a_init.shape != (dims[mode], factors.rank):
        raise InvalidArgument("s_nmc: a_init shape mismatch")
    if not np.all(a_init >= 0):
        raise InvalidArgument("s_nmc: a_init must be nonnegative")
    _push_factors(t, factors)
    acc = t.ctx.s_nmc(mode, cfg, rng.state, a_init)
    a, y = t.ctx.get_factor(mode)
    factors.factors[mode] = a
    factors.momentum[mode] = y
    if stats is not None:
        stats.entries_accessed += acc
    return factors.factors[mode]


def objective(t: SparseTensor, factors: FactorSet, lam: float) -> float:
    if factors.order() != t.order() or any(
            u.shape != (d, factors.rank) for u, d in zip(factors.factors, t.dims())):
        raise InvalidArgument("objective: factor shapes do not match tensor")
    if lam < 0.0:
        raise InvalidArgument("objective: lambda must be >= 0")
    _push_factors(t, factors)
    return t.ctx.objective(lam)


def relative_error(t: SparseTensor, factors: FactorSet) -> float:
    if factors.order() != t.order() or any(
            u.shape != (d, factors.rank) for u, d in zip(factors.factors, t.dims())):
        raise InvalidArgument("relative_error: factor shapes do not match tensor")
    _push_factors(t, factors)
    return t.ctx.relative_error()


@dataclass
class AoResult:
    factors: FactorSet
    history: List[MetricsRecord]


def ao_ntc(t: SparseTensor, init: FactorSet, cfg: AoConfig,
           observer: Optional[Callable[[MetricsRecord, FactorSet], None]] = None) -> AoResult:
    """ntc::ao_ntc (ao.cpp:75-133); the loop runs inside libntcb (ntcb_ao_ntc)."""
    cfg.validate()
    if init.rank != cfg.rank:
        raise InvalidArgument("ao_ntc: init rank differs from configured rank")
    if init.order() != t.order() or any(
            u.shape != (d, init.rank) for u, d in zip(init.factors, t.dims())):
        raise InvalidArgument("ao_ntc: init factor shapes do not match tensor")
    if not init.all_nonnegative():
        raise InvalidArgument("ao_ntc: init factors must be nonnegative")
    _push_factors(t, init)

    def _pull():
        f = FactorSet(init.rank, [], [])
        for m in range(t.order()):
            a, y = t.ctx.get_factor(m)
            f.factors.append(a)
            f.momentum.append(y)
        return f

    obs = None
    if observer is not None:
        def obs(rec):
            observer(rec, _pull())
    hist = t.ctx.ao_ntc(cfg, obs)
    return AoResult(_pull(), hist)
