"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the ntc hot path.

Two numpy-facing wrappers:

* ``Oracle``  — the plain-C restatement ``oracle/ntc_oracle.c`` (always built).
* ``RefProblem`` / ``ref_lib()`` — the UNMODIFIED reference library compiled
  from /root/reference by ``oracle/Makefile`` into ``oracle/_ref/libntc_ref.so``
  (present wherever ``make -C oracle`` ran with the reference mounted; the
  gpurun snapshot carries the built .so to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference``) may import this package, and only as the checker or
the timed reference arm — never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libntc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libntc_ref.so")

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)

_EXC = {1: ValueError, 2: RuntimeError, 3: IndexError, 4: ArithmeticError, 5: RuntimeError}


class OracleError(Exception):
    pass


def build(quiet: bool = True) -> None:
    """Compile oracle/ (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _arr_ptrs(arrs, t):
    ptrs = (t * len(arrs))()
    for i, a in enumerate(arrs):
        ptrs[i] = a.ctypes.data_as(t)
    return ptrs


class NmcCfg(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("c", C.c_double), ("max_inner", C.c_int),
                ("power_iters", C.c_int), ("power_tol", C.c_double), ("threads", C.c_int),
                ("chunk", C.c_int)]


class AoCfg(C.Structure):
    _fields_ = [("rank", C.c_uint64), ("lambda_", C.c_double), ("c", C.c_double),
                ("max_inner", C.c_int), ("max_epochs", C.c_double), ("term_tol", C.c_double),
                ("seed", C.c_uint64), ("threads", C.c_int), ("chunk", C.c_int),
                ("power_iters", C.c_int), ("power_tol", C.c_double), ("eval_metrics", C.c_int),
                ("metrics_every", C.c_int)]


def nmc_cfg(lambda_=1e-3, c=1.0, max_inner=1, power_iters=30, power_tol=1e-6, threads=1, chunk=0):
    return NmcCfg(lambda_, c, max_inner, power_iters, power_tol, threads, chunk)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_fork.restype = C.c_uint64
        L.orc_fork.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_sweep_state.restype = C.c_uint64
        L.orc_sweep_state.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.orc_blocksize.restype = C.c_uint64
        L.orc_blocksize.argtypes = [C.c_double, C.c_uint64]
        L.orc_next_u64_n.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.orc_next_double_n.argtypes = [C.c_uint64, C.c_int, _f64p]
        L.orc_next_below_n.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _u64p]
        L.orc_sample_row.restype = C.c_uint64
        L.orc_sample_row.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _u32p]
        L.orc_canonicalize.argtypes = [C.c_int, _u64p, C.c_uint64, _u32p, _f64p, _u32p, _f64p]
        L.orc_build_view.argtypes = [C.c_int, _u64p, C.c_uint64, _u32p, _f64p, C.c_int, _u64p,
                                     _u32p, _f64p]
        L.orc_power_method.argtypes = [C.c_uint64, _f64p, C.c_int, C.c_double, _f64p]
        L.orc_row_step.argtypes = [C.c_uint64, _f64p, _f64p, _f64p, C.c_double, C.c_double, _f64p,
                                   _f64p, _f64p]
        L.orc_row_terms.argtypes = [C.c_int, _u64p, C.c_uint64, C.POINTER(_f64p), C.c_int, _u64p,
                                    _u32p, _f64p, C.c_uint64, _u32p, C.c_uint64, _f64p, C.c_double,
                                    _f64p, _f64p, _f64p, _f64p]
        L.orc_s_nmc.argtypes = [C.c_int, _u64p, C.c_uint64, C.POINTER(_f64p), C.POINTER(_f64p),
                                C.c_int, _u64p, _u32p, _f64p, _f64p, C.POINTER(NmcCfg),
                                C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.orc_metrics.argtypes = [C.c_int, _u64p, C.c_uint64, C.POINTER(_f64p), C.c_uint64, _u32p,
                                  _f64p, _f64p, _f64p, _f64p]
        L.orc_objective.argtypes = [C.c_int, _u64p, C.c_uint64, C.POINTER(_f64p), C.c_uint64,
                                    _u32p, _f64p, C.c_double, _f64p]
        L.orc_relative_error.argtypes = [C.c_int, _u64p, C.c_uint64, C.POINTER(_f64p), C.c_uint64,
                                         _u32p, _f64p, _f64p]
        L.orc_initial_factors.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_uint64, _f64p]
        L.orc_sample_mask_rows.argtypes = [C.c_uint64, _u64p, C.c_double, C.c_uint64,
                                           C.POINTER(C.c_uint8), C.c_int]
        L.ntco_synth.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, _f64p,
                                 C.c_int, C.c_int, C.c_int, _u32p, C.POINTER(C.c_float)]

    def _check(self, rc):
        if rc:
            raise _EXC.get(rc, RuntimeError)(self.L.orc_last_error().decode())

    # RNG
    def mix(self, z): return self.L.orc_mix(z)
    def fork(self, s, t): return self.L.orc_fork(s, t)
    def sweep_state(self, seed, k, mode): return self.L.orc_sweep_state(seed, k, mode)
    def blocksize(self, c, n): return self.L.orc_blocksize(c, n)

    def next_u64(self, state, n):
        out = np.zeros(n, np.uint64)
        self.L.orc_next_u64_n(state, n, _ptr(out, _u64p))
        return out

    def next_double(self, state, n):
        out = np.zeros(n, np.float64)
        self.L.orc_next_double_n(state, n, _ptr(out, _f64p))
        return out

    def next_below(self, state, bound, n):
        out = np.zeros(n, np.uint64)
        self.L.orc_next_below_n(state, bound, n, _ptr(out, _u64p))
        return out

    def sample_row(self, n, c, state):
        picks = np.zeros(max(n, 1), np.uint32)
        b = self.L.orc_sample_row(n, c, state, _ptr(picks, _u32p))
        return picks[:b].copy()

    def sample_mask_rows(self, off, c, root, threads=None):
        """Per-entry 0/1 array of the sampled sets of every row of a view
        (row streams fork(root, p)), computed on the host cores."""
        off = np.ascontiguousarray(off, np.uint64)
        out = np.zeros(max(int(off[-1]), 1), np.uint8)
        self.L.orc_sample_mask_rows(len(off) - 1, _ptr(off, _u64p), c, root,
                                    out.ctypes.data_as(C.POINTER(C.c_uint8)), threads or os.cpu_count() or 1)
        return out[: int(off[-1])]

    # tensor / views
    def canonicalize(self, dims, idx, vals):
        dims = np.ascontiguousarray(dims, np.uint64)
        idx = np.ascontiguousarray(idx, np.uint32).reshape(-1)
        vals = np.ascontiguousarray(vals, np.float64)
        oi, ov = np.empty_like(idx), np.empty_like(vals)
        self._check(self.L.orc_canonicalize(len(dims), _ptr(dims, _u64p), len(vals),
                                            _ptr(idx, _u32p), _ptr(vals, _f64p),
                                            _ptr(oi, _u32p), _ptr(ov, _f64p)))
        return oi.reshape(len(vals), len(dims)), ov

    def build_view(self, dims, idx_c, vals_c, mode):
        dims = np.ascontiguousarray(dims, np.uint64)
        N = len(dims)
        idx_c = np.ascontiguousarray(idx_c, np.uint32).reshape(-1)
        vals_c = np.ascontiguousarray(vals_c, np.float64)
        nnz = len(vals_c)
        off = np.zeros(int(dims[mode]) + 1, np.uint64)
        oth = np.zeros(max(nnz * (N - 1), 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        self.L.orc_build_view(N, _ptr(dims, _u64p), nnz, _ptr(idx_c, _u32p), _ptr(vals_c, _f64p),
                              mode, _ptr(off, _u64p), _ptr(oth, _u32p), _ptr(val, _f64p))
        return off, oth[: nnz * (N - 1)].reshape(nnz, N - 1), val[:nnz]

    # numerics
    def power_method(self, H, iters=30, tol=1e-6):
        H = np.ascontiguousarray(H, np.float64)
        out = C.c_double()
        self._check(self.L.orc_power_method(H.shape[0], _ptr(H, _f64p), iters, tol, C.byref(out)))
        return out.value

    def row_step(self, y, a_prev, grad, L, lam):
        y, a_prev, grad = (np.ascontiguousarray(v, np.float64) for v in (y, a_prev, grad))
        a_new, y_new = np.zeros_like(y), np.zeros_like(y)
        beta = C.c_double()
        self._check(self.L.orc_row_step(len(y), _ptr(y, _f64p), _ptr(a_prev, _f64p),
                                        _ptr(grad, _f64p), L, lam, _ptr(a_new, _f64p),
                                        _ptr(y_new, _f64p), C.byref(beta)))
        return a_new, y_new, beta.value

    def s_nmc(self, dims, rank, factors, momentum, mode, view, a_init, cfg, rng_state,
              row_begin=0, row_end=None):
        """factors/momentum: lists of float64 (I_m, R) arrays, updated in place
        on rows [row_begin, row_end) of `mode`.  Returns entries accessed."""
        dims = np.ascontiguousarray(dims, np.uint64)
        off, oth, val = view
        off = np.ascontiguousarray(off, np.uint64)
        oth = np.ascontiguousarray(oth, np.uint32).reshape(-1)
        val = np.ascontiguousarray(val, np.float64)
        if oth.size == 0:
            oth = np.zeros(1, np.uint32)
        if val.size == 0:
            val = np.zeros(1, np.float64)
        if row_end is None:
            row_end = int(dims[mode])
        for f in list(factors) + list(momentum):
            assert f.dtype == np.float64 and f.flags.c_contiguous
        fp = _arr_ptrs(factors, _f64p)
        mp = _arr_ptrs(momentum, _f64p)
        a_init = factors[mode] if a_init is None else np.ascontiguousarray(a_init, np.float64)
        acc = C.c_uint64(0)
        self._check(self.L.orc_s_nmc(len(dims), _ptr(dims, _u64p), rank, fp, mp, mode,
                                     _ptr(off, _u64p), _ptr(oth, _u32p), _ptr(val, _f64p),
                                     _ptr(a_init, _f64p), C.byref(cfg), rng_state, row_begin,
                                     row_end, C.byref(acc)))
        return acc.value

    def metrics(self, dims, rank, factors, idx_c, vals_c):
        dims = np.ascontiguousarray(dims, np.uint64)
        idx_c = np.ascontiguousarray(idx_c, np.uint32).reshape(-1)
        vals_c = np.ascontiguousarray(vals_c, np.float64)
        fp = _arr_ptrs(factors, _f64p)
        sse, den, reg = C.c_double(), C.c_double(), C.c_double()
        self.L.orc_metrics(len(dims), _ptr(dims, _u64p), rank, fp, len(vals_c), _ptr(idx_c, _u32p),
                           _ptr(vals_c, _f64p), C.byref(sse), C.byref(den), C.byref(reg))
        return sse.value, den.value, reg.value

    def initial_factors(self, dims, rank, seed):
        dims = np.ascontiguousarray(dims, np.uint64)
        out = np.zeros(int(dims.sum()) * rank, np.float64)
        self.L.orc_initial_factors(len(dims), _ptr(dims, _u64p), rank, seed, _ptr(out, _f64p))
        res, pos = [], 0
        for d in dims:
            res.append(out[pos: pos + int(d) * rank].reshape(int(d), rank).copy())
            pos += int(d) * rank
        return res


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref/libntc_ref.so)
# --------------------------------------------------------------------------
_REF = None


def host_synth(dims, nnz, true_rank, sigma, seed, zipf_alpha=None, value_kind=0, canonical=False,
               threads=None):
    """The repo's synthetic tensor generated on the host cores
    (oracle/synth_host.c, a C restatement of csrc/synth.cu, bit-identical):
    (indices (nnz, N) uint32, values float32), in generation order (what the
    device canonicalises) or, with canonical=True, lexicographic order."""
    L = Oracle().L
    N = len(dims)
    d = np.ascontiguousarray(dims, np.uint64)
    z = None if zipf_alpha is None else np.ascontiguousarray(zipf_alpha, np.float64)
    idx = np.empty(max(nnz * N, 1), np.uint32)
    vals = np.empty(max(nnz, 1), np.float32)
    rc = L.ntco_synth(N, _ptr(d, _u64p), nnz, true_rank, sigma, seed, _ptr(z, _f64p), value_kind,
                      1 if canonical else 0, threads or os.cpu_count() or 1,
                      _ptr(idx, _u32p), vals.ctypes.data_as(C.POINTER(C.c_float)))
    if rc:
        raise ValueError({1: "host_synth: invalid configuration", 2: "host_synth: too many candidates",
                          3: "host_synth: out of memory"}.get(rc, f"host_synth: error {rc}"))
    return idx[: nnz * N].reshape(nnz, N), vals[:nnz]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _REF
    if _REF is None:
        if not os.path.exists(REF_SO):
            raise OracleError("oracle/_ref/libntc_ref.so not built (needs /root/reference)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_next_u64.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.ref_rng_next_double.argtypes = [C.c_uint64, C.c_int, _f64p]
        L.ref_rng_next_below.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _u64p]
        L.ref_rng_fork_first.restype = C.c_uint64
        L.ref_rng_fork_first.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_row_stream_first.restype = C.c_uint64
        L.ref_row_stream_first.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64]
        L.ref_mix.restype = C.c_uint64
        L.ref_mix.argtypes = [C.c_uint64]
        L.ref_tensor_new.restype = C.c_void_p
        L.ref_tensor_new.argtypes = [C.c_int, _u64p, C.c_uint64, _u32p, _f64p]
        L.ref_views_new.restype = C.c_void_p
        L.ref_views_new.argtypes = [C.c_int, _u64p, _u64p, C.POINTER(_u64p), C.POINTER(_u32p),
                                    C.POINTER(_f64p)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_nnz.restype = C.c_uint64
        L.ref_nnz.argtypes = [C.c_void_p]
        L.ref_tensor_export.argtypes = [C.c_void_p, _u32p, _f64p]
        L.ref_view_rows.restype = C.c_uint64
        L.ref_view_rows.argtypes = [C.c_void_p, C.c_int]
        L.ref_view_nnz.restype = C.c_uint64
        L.ref_view_nnz.argtypes = [C.c_void_p, C.c_int]
        L.ref_view_export.argtypes = [C.c_void_p, C.c_int, _u64p, _u32p, _f64p]
        L.ref_sample_row.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_uint64, _u32p,
                                     _u64p]
        L.ref_factors_init.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_f64p), C.POINTER(_f64p)]
        L.ref_factor_resize.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _f64p]
        L.ref_factors_get.argtypes = [C.c_void_p, C.c_int, _f64p, _f64p]
        L.ref_s_nmc.argtypes = [C.c_void_p, C.c_int, _f64p, C.c_uint64, C.POINTER(NmcCfg),
                                C.c_uint64, _u64p]
        L.ref_objective.argtypes = [C.c_void_p, C.c_double, _f64p]
        L.ref_relative_error.argtypes = [C.c_void_p, _f64p]
        L.ref_initial_factors.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_uint64, _f64p]
        L.ref_ao_ntc.argtypes = [C.c_void_p, C.POINTER(AoCfg), _f64p, _f64p, _f64p, C.c_int,
                                 C.POINTER(C.c_int)]
        L.ref_power_method.argtypes = [C.c_uint64, _f64p, C.c_int, C.c_double, _f64p]
        L.ref_render_model.argtypes = [C.c_int, _u64p, C.c_uint64, C.POINTER(_f64p), C.POINTER(C.c_uint8)]
        L.ref_row_step.argtypes = [C.c_uint64, _f64p, _f64p, _f64p, C.c_double, C.c_double, _f64p,
                                   _f64p, _f64p]
        L.ref_row_terms.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _u32p, C.c_uint64, _f64p,
                                    C.c_double, _f64p, _f64p, _f64p, _f64p]
        L.ref_read_tns.restype = C.c_void_p
        L.ref_read_tns.argtypes = [C.c_char_p]
        L.ref_order.restype = C.c_int
        L.ref_order.argtypes = [C.c_void_p]
        L.ref_dims.argtypes = [C.c_void_p, _u64p]
        L.ref_write_tns.argtypes = [C.c_void_p, C.c_char_p]
        _REF = L
    return _REF


def ref_read_tns(path):
    """The reference's read_tns: (dims, canonical idx, vals) or raises with its message."""
    L = ref_lib()
    h = L.ref_read_tns(path.encode())
    if not h:
        raise RuntimeError(L.ref_last_error().decode())
    p = RefProblem.__new__(RefProblem)
    p.h = C.c_void_p(h)
    p.rank = None
    N = L.ref_order(p.h)
    d = np.zeros(N, np.uint64)
    L.ref_dims(p.h, _ptr(d, _u64p))
    p.dims = d
    return p


def _ref_check(rc):
    if rc:
        raise _EXC.get(rc, RuntimeError)(ref_lib().ref_last_error().decode())


def ref_rng(state, n, kind="u64", bound=None):
    L = ref_lib()
    if kind == "u64":
        out = np.zeros(n, np.uint64)
        L.ref_rng_next_u64(state, n, _ptr(out, _u64p))
    elif kind == "double":
        out = np.zeros(n, np.float64)
        L.ref_rng_next_double(state, n, _ptr(out, _f64p))
    else:
        out = np.zeros(n, np.uint64)
        L.ref_rng_next_below(state, bound, n, _ptr(out, _u64p))
    return out


def ref_initial_factors(dims, rank, seed):
    dims = np.ascontiguousarray(dims, np.uint64)
    out = np.zeros(int(dims.sum()) * rank, np.float64)
    _ref_check(ref_lib().ref_initial_factors(len(dims), _ptr(dims, _u64p), rank, seed,
                                             _ptr(out, _f64p)))
    res, pos = [], 0
    for d in dims:
        res.append(out[pos: pos + int(d) * rank].reshape(int(d), rank).copy())
        pos += int(d) * rank
    return res


def ref_render_model(factors):
    """The reference's render_model (image.cpp:161-183): (H, W, 3) uint8."""
    fs = [np.ascontiguousarray(f, np.float64) for f in factors]
    dims = np.array([f.shape[0] for f in fs], np.uint64)
    R = fs[0].shape[1]
    H, W = int(dims[0]), int(dims[1])
    out = np.zeros(max(3 * H * W, 1), np.uint8)
    _ref_check(ref_lib().ref_render_model(len(fs), _ptr(dims, _u64p), R, _arr_ptrs(fs, _f64p),
                                          out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out[: 3 * H * W].reshape(H, W, 3)


def ref_power_method(H, iters=30, tol=1e-6):
    H = np.ascontiguousarray(H, np.float64)
    out = C.c_double()
    _ref_check(ref_lib().ref_power_method(H.shape[0], _ptr(H, _f64p), iters, tol, C.byref(out)))
    return out.value


def ref_row_step(y, a_prev, grad, L, lam):
    y, a_prev, grad = (np.ascontiguousarray(v, np.float64) for v in (y, a_prev, grad))
    a_new, y_new = np.zeros_like(y), np.zeros_like(y)
    beta = C.c_double()
    _ref_check(ref_lib().ref_row_step(len(y), _ptr(y, _f64p), _ptr(a_prev, _f64p),
                                      _ptr(grad, _f64p), L, lam, _ptr(a_new, _f64p),
                                      _ptr(y_new, _f64p), C.byref(beta)))
    return a_new, y_new, beta.value


class RefProblem:
    """A reference SparseTensor + its mode views (+ optional FactorSet)."""

    def __init__(self, dims, idx=None, vals=None, views=None):
        L = ref_lib()
        self.dims = np.ascontiguousarray(dims, np.uint64)
        N = len(self.dims)
        if views is None:
            idx = np.ascontiguousarray(idx, np.uint32).reshape(-1)
            vals = np.ascontiguousarray(vals, np.float64)
            if idx.size == 0:
                idx = np.zeros(1, np.uint32)
            if vals.size == 0:
                nnz = 0
                vals = np.zeros(1, np.float64)
            else:
                nnz = len(vals)
            h = L.ref_tensor_new(N, _ptr(self.dims, _u64p), nnz, _ptr(idx, _u32p), _ptr(vals, _f64p))
        else:
            # views: list of (offsets, others, values) per mode (row-prefix samples allowed)
            self._keep = [tuple(np.ascontiguousarray(a) for a in v) for v in views]
            rows = np.array([len(v[0]) - 1 for v in self._keep], np.uint64)
            offs = _arr_ptrs([np.ascontiguousarray(v[0], np.uint64) for v in self._keep], _u64p)
            oths = _arr_ptrs([np.ascontiguousarray(v[1], np.uint32).reshape(-1) for v in self._keep], _u32p)
            vls = _arr_ptrs([np.ascontiguousarray(v[2], np.float64) for v in self._keep], _f64p)
            self._rows = rows
            h = L.ref_views_new(N, _ptr(self.dims, _u64p), _ptr(rows, _u64p), offs, oths, vls)
        if not h:
            raise ValueError(L.ref_last_error().decode())
        self.h = C.c_void_p(h)
        self.rank = None

    def __del__(self):
        try:
            ref_lib().ref_free(self.h)
        except Exception:
            pass

    @property
    def nnz(self):
        return ref_lib().ref_nnz(self.h)

    def tensor(self):
        N, nnz = len(self.dims), self.nnz
        idx = np.zeros(max(nnz * N, 1), np.uint32)
        vals = np.zeros(max(nnz, 1), np.float64)
        _ref_check(ref_lib().ref_tensor_export(self.h, _ptr(idx, _u32p), _ptr(vals, _f64p)))
        return idx[: nnz * N].reshape(nnz, N), vals[:nnz]

    def view(self, mode):
        L = ref_lib()
        N = len(self.dims)
        rows = L.ref_view_rows(self.h, mode)
        nnz = L.ref_view_nnz(self.h, mode)
        off = np.zeros(rows + 1, np.uint64)
        oth = np.zeros(max(nnz * (N - 1), 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        _ref_check(L.ref_view_export(self.h, mode, _ptr(off, _u64p), _ptr(oth, _u32p), _ptr(val, _f64p)))
        return off, oth[: nnz * (N - 1)].reshape(nnz, N - 1), val[:nnz]

    def sample_row(self, mode, row, c, state):
        L = ref_lib()
        rows = L.ref_view_rows(self.h, mode)
        n = self.view(mode)[0]
        cap = int(n[row + 1] - n[row]) if row < rows else 1
        picks = np.zeros(max(cap, 1), np.uint32)
        cnt = C.c_uint64()
        _ref_check(L.ref_sample_row(self.h, mode, row, c, state, _ptr(picks, _u32p), C.byref(cnt)))
        return picks[: cnt.value].copy()

    def set_factors(self, rank, factors, momentum=None):
        self.rank = rank
        fs = [np.ascontiguousarray(f, np.float64) for f in factors]
        ms = [np.ascontiguousarray(f, np.float64) for f in momentum] if momentum is not None else None
        self._fs = (fs, ms)
        _ref_check(ref_lib().ref_factors_init(self.h, rank, _arr_ptrs(fs, _f64p),
                                              _arr_ptrs(ms, _f64p) if ms else None))

    def set_factor_rows(self, mode, a):
        a = np.ascontiguousarray(a, np.float64)
        _ref_check(ref_lib().ref_factor_resize(self.h, mode, a.shape[0], _ptr(a, _f64p)))

    def get_factor(self, mode, rows=None):
        rows = int(self.dims[mode]) if rows is None else rows
        a = np.zeros((rows, self.rank), np.float64)
        y = np.zeros((rows, self.rank), np.float64)
        _ref_check(ref_lib().ref_factors_get(self.h, mode, _ptr(a, _f64p), _ptr(y, _f64p)))
        return a, y

    def s_nmc(self, mode, cfg, rng_state, a_init=None):
        acc = C.c_uint64(0)
        if a_init is not None:
            a_init = np.ascontiguousarray(a_init, np.float64)
            rows = a_init.shape[0]
        else:
            rows = 0
        _ref_check(ref_lib().ref_s_nmc(self.h, mode, _ptr(a_init, _f64p), rows, C.byref(cfg),
                                       rng_state, C.byref(acc)))
        return acc.value

    def objective(self, lam):
        out = C.c_double()
        _ref_check(ref_lib().ref_objective(self.h, lam, C.byref(out)))
        return out.value

    def relative_error(self):
        out = C.c_double()
        _ref_check(ref_lib().ref_relative_error(self.h, C.byref(out)))
        return out.value

    def row_terms(self, mode, row, picks, y, lam):
        R = self.rank
        picks = np.ascontiguousarray(picks, np.uint32)
        if picks.size == 0:
            picks = np.zeros(1, np.uint32)
            npk = 0
        else:
            npk = len(picks)
        y = np.ascontiguousarray(y, np.float64)
        w, z, g = (np.zeros(R) for _ in range(3))
        H = np.zeros((R, R))
        _ref_check(ref_lib().ref_row_terms(self.h, mode, row, _ptr(picks, _u32p), npk,
                                           _ptr(y, _f64p), lam, _ptr(w, _f64p), _ptr(z, _f64p),
                                           _ptr(g, _f64p), _ptr(H, _f64p)))
        return w, z, g, H

    def ao_ntc(self, init, rank, lambda_=1e-3, c=1.0, max_inner=1, max_epochs=100.0,
               term_tol=0.0, seed=0, threads=1, chunk=0, power_iters=30, power_tol=1e-6,
               eval_metrics=True, metrics_every=1, max_hist=100000):
        cfg = AoCfg(rank, lambda_, c, max_inner, max_epochs, term_tol, seed, threads, chunk,
                    power_iters, power_tol, int(eval_metrics), metrics_every)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(f, np.float64).reshape(-1) for f in init]))
        out = np.zeros_like(flat)
        hist = np.zeros(max_hist * 5, np.float64)
        nh = C.c_int()
        _ref_check(ref_lib().ref_ao_ntc(self.h, C.byref(cfg), _ptr(flat, _f64p), _ptr(out, _f64p),
                                        _ptr(hist, _f64p), max_hist, C.byref(nh)))
        res, pos = [], 0
        for d in self.dims:
            res.append(out[pos: pos + int(d) * rank].reshape(int(d), rank).copy())
            pos += int(d) * rank
        return res, hist[: 5 * min(nh.value, max_hist)].reshape(-1, 5)
