"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle and the compiled reference.

``Oracle``    wraps ``oracle/liboracle.so`` (our plain-C restatement, oracle.c).
``Reference`` wraps ``oracle/_ref/libmttkrp_ref.so`` (the reference library compiled from
              /root/reference sources by oracle/Makefile; travels prebuilt to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference arm may
import this package, and only as the checker or the CPU baseline.  The product package
``paper_2503_18198_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    pass


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when the reference sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _dims(dims):
    return np.ascontiguousarray(np.asarray(dims, dtype=np.uint32))


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(self.path)
        self.lib = C.CDLL(self.path)
        # attribute access caches the function object (lib[...] builds a new one per call)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            raise OracleError(getattr(self.lib, self.prefix + "last_error")().decode())

    def random_factors(self, dims, rank, seed):
        dims = _dims(dims)
        total = int(sum(int(d) for d in dims)) * rank
        out = np.empty(total, dtype=np.float32)
        f = self.lib[self.prefix + "random_factors"]
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_uint64, _f32p]
        self._check(f(len(dims), dims, rank, seed, out))
        mats, off = [], 0
        for d in dims:
            mats.append(out[off:off + int(d) * rank].reshape(int(d), rank))
            off += int(d) * rank
        return mats

    def generate_synthetic(self, dims, nnz, dist=0, skew_mode=0, skew_distinct=2, seed=0):
        dims = _dims(dims)
        coords = np.empty(nnz * len(dims), dtype=np.uint32)
        vals = np.empty(nnz, dtype=np.float32)
        f = self.lib[self.prefix + "generate_synthetic"]
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                      C.c_uint64, _u32p, _f32p]
        self._check(f(len(dims), dims, nnz, dist, skew_mode, skew_distinct, seed, coords, vals))
        return coords.reshape(nnz, len(dims)), vals

    def build_plan(self, dims, coords, mode, kappa, strategy=0, policy=0, values=None):
        dims = _dims(dims)
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        order = np.empty(max(nnz, 1), dtype=np.uint64)
        offsets = np.empty(kappa + 1, dtype=np.uint64)
        owned = np.empty(int(dims[mode]) + 1, dtype=np.uint32)
        owned_off = np.empty(kappa + 1, dtype=np.uint64)
        scheme = C.c_int(0)
        f = self.lib[self.prefix + "build_plan"]
        if self.prefix == "ref_":
            if values is None:
                values = np.ones(nnz, dtype=np.float32)
            f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint32, C.c_uint64,
                          C.c_int, C.c_int, _ip, _u64p, _u64p, _u32p, _u64p]
            rc = f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, dtype=np.float32),
                   mode, kappa, strategy, policy, C.byref(scheme), order, offsets, owned,
                   owned_off)
        else:
            f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, C.c_uint32, C.c_uint64,
                          C.c_int, C.c_int, _ip, _u64p, _u64p, _u32p, _u64p]
            rc = f(len(dims), dims, nnz, coords, mode, kappa, strategy, policy,
                   C.byref(scheme), order, offsets, owned, owned_off)
        self._check(rc)
        return {"scheme": scheme.value, "order": order[:nnz], "offsets": offsets,
                "owned": owned[:int(owned_off[-1])], "owned_offsets": owned_off}

    def _factor_concat(self, factors):
        return np.ascontiguousarray(np.concatenate([np.asarray(f, np.float32).reshape(-1)
                                                    for f in factors]))


class Oracle(_Lib):
    """Our C restatement (oracle/oracle.c)."""
    prefix = "orc_"
    path = os.path.join(HERE, "liboracle.so")

    def generate_powerlaw(self, dims, nnz, exponent=1.0, seed=0):
        dims = _dims(dims)
        coords = np.empty(nnz * len(dims), dtype=np.uint32)
        vals = np.empty(nnz, dtype=np.float32)
        f = self.lib.orc_generate_powerlaw
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_double, C.c_uint64, _u32p, _f32p]
        self._check(f(len(dims), dims, nnz, exponent, seed, coords, vals))
        return coords.reshape(nnz, len(dims)), vals

    def mttkrp(self, dims, coords, values, factors, mode):
        dims = _dims(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        out = np.empty(int(dims[mode]) * rank, dtype=np.float32)
        f = self.lib.orc_mttkrp
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p,
                      C.c_uint32, _f32p]
        self._check(f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, np.float32),
                      rank, self._factor_concat(factors), mode, out))
        return out.reshape(int(dims[mode]), rank)

    def mttkrp_f64(self, dims, coords, values, factors, mode, threads=None):
        """oracle.hpp:20-43 with T = double (row-parallel, bitwise = the reference's fp64)."""
        dims = _dims(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        out = np.empty(int(dims[mode]) * rank, dtype=np.float64)
        f = self.lib.orc_mttkrp_f64
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p,
                      C.c_uint32, _f64p, C.c_uint32]
        self._check(f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, np.float32),
                      rank, self._factor_concat(factors), mode, out,
                      int(threads or os.cpu_count() or 1)))
        return out.reshape(int(dims[mode]), rank)

    def max_rel_err_f64(self, got, want):
        g = np.ascontiguousarray(got, dtype=np.float32).reshape(-1)
        w = np.ascontiguousarray(want, dtype=np.float64).reshape(-1)
        assert g.size == w.size
        f = self.lib.orc_max_rel_err_f64
        f.argtypes = [_f32p, _f64p, C.c_uint64]
        f.restype = C.c_double
        return float(f(g, w, g.size))

    def build_plans_all(self, dims, coords, kappa, strategy=0, policy=0):
        """Every mode's plan, in the array layout of Reference.run_timed_plans."""
        return [self.build_plan(dims, coords, d, kappa, strategy, policy)
                for d in range(len(dims))]

    def max_rel_err(self, got, want):
        g = np.ascontiguousarray(got, dtype=np.float32).reshape(-1)
        w = np.ascontiguousarray(want, dtype=np.float32).reshape(-1)
        assert g.size == w.size
        f = self.lib.orc_max_rel_err
        f.argtypes = [_f32p, _f32p, C.c_uint64]
        f.restype = C.c_double
        return float(f(g, w, g.size))


class Reference(_Lib):
    """The unmodified reference compiled from /root/reference (oracle/_ref)."""
    prefix = "ref_"
    path = os.path.join(HERE, "_ref", "libmttkrp_ref.so")

    def oracle_mttkrp(self, dims, coords, values, factors, mode):
        dims = _dims(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        out = np.empty(int(dims[mode]) * rank, dtype=np.float32)
        f = self.lib.ref_oracle_mttkrp
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p,
                      C.c_uint32, _f32p]
        self._check(f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, np.float32),
                      rank, self._factor_concat(factors), mode, out))
        return out.reshape(int(dims[mode]), rank)

    def oracle_mttkrp_f64(self, dims, coords, values, factors, mode):
        """oracle_mttkrp<double> (oracle.hpp:20-43) on the fp32 inputs widened to double."""
        dims = _dims(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        out = np.empty(int(dims[mode]) * rank, dtype=np.float64)
        f = self.lib.ref_oracle_mttkrp_f64
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p,
                      C.c_uint32, _f64p]
        self._check(f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, np.float32),
                      rank, self._factor_concat(factors), mode, out))
        return out.reshape(int(dims[mode]), rank)

    def build_plans_all(self, dims, coords, values, kappa, strategy=0, policy=0):
        """build_mode_plans once; every mode exported (list of dicts like build_plan) plus
        the reference's plan-build wall time (ms)."""
        dims = _dims(dims)
        n = len(dims)
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // n
        schemes = np.zeros(n, dtype=np.int32)
        orders = np.empty(max(n * nnz, 1), dtype=np.uint64)
        offsets = np.empty(n * (kappa + 1), dtype=np.uint64)
        owned = np.empty(int(sum(int(d) for d in dims)) + 1, dtype=np.uint32)
        owned_off = np.empty(n * (kappa + 1), dtype=np.uint64)
        plan_ms = C.c_double(0)
        f = self.lib.ref_build_plans_all
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, C.c_int, C.c_int,
                      np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"), _u64p,
                      _u64p, _u32p, _u64p, C.POINTER(C.c_double)]
        self._check(f(n, dims, nnz, coords, np.ascontiguousarray(values, np.float32), kappa,
                      strategy, policy, schemes, orders, offsets, owned, owned_off,
                      C.byref(plan_ms)))
        plans, base = [], 0
        for d in range(n):
            oo = owned_off[d * (kappa + 1):(d + 1) * (kappa + 1)]
            plans.append({"scheme": int(schemes[d]), "order": orders[d * nnz:(d + 1) * nnz],
                          "offsets": offsets[d * (kappa + 1):(d + 1) * (kappa + 1)],
                          "owned": owned[base:base + int(oo[-1])], "owned_offsets": oo})
            base += int(dims[d])
        return plans, plan_ms.value

    def frostt_parse(self, text, prec=32, merge=True, dims_override=None, max_modes=16):
        """parse_frostt<T> (frostt.hpp:74-160): (dims, coords, values, duplicates_merged)."""
        raw = text.encode() if isinstance(text, str) else bytes(text)
        cap = raw.count(b"\n") + 1
        ovr = np.asarray(dims_override if dims_override else [0], dtype=np.uint32)
        n, nnz, dups = C.c_uint32(), C.c_uint64(), C.c_uint64()
        dims = np.zeros(max_modes, dtype=np.uint32)
        coords = np.empty(cap * max_modes, dtype=np.uint32)
        vals = np.empty(cap, dtype=np.float64 if prec == 64 else np.float32)
        f = self.lib.ref_frostt_parse
        f.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_uint32,
                      C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32), C.c_void_p,
                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p]
        self._check(f(raw, len(raw), prec, 1 if merge else 0, ovr.ctypes.data,
                      len(dims_override) if dims_override else 0, cap, max_modes,
                      C.byref(n), dims.ctypes.data, C.byref(nnz), C.byref(dups),
                      coords.ctypes.data, vals.ctypes.data))
        k, m = n.value, nnz.value
        return (dims[:k].tolist(), coords[:m * k].reshape(m, k).copy(), vals[:m].copy(),
                dups.value)

    def frostt_write(self, dims, coords, values):
        """write_frostt_string (frostt.hpp:165-192) of a tensor (fp32 or fp64 values)."""
        dims = _dims(dims)
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        prec = 64 if np.asarray(values).dtype == np.float64 else 32
        values = np.ascontiguousarray(values, dtype=np.float64 if prec == 64 else np.float32)
        nnz = values.size
        cap = nnz * (len(dims) * 11 + 32) + 1
        out = C.create_string_buffer(cap)
        ln = C.c_uint64()
        f = self.lib.ref_frostt_write
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int,
                      C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
        self._check(f(len(dims), dims, nnz, coords.ctypes.data, values.ctypes.data, prec, out,
                      cap, C.byref(ln)))
        return out.raw[:ln.value].decode()

    def run_timed_plans(self, dims, coords, values, factors, kappa, plans, iters, batch_p=32):
        """The reference's run_timed (kernel.hpp:239-287) on given plans (list of build_plan
        dicts).  Returns (total_ms per iteration, per-mode min ms, outputs_bit_identical)."""
        dims = _dims(dims)
        n = len(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // n
        schemes = np.array([p["scheme"] for p in plans], dtype=np.int32)
        orders = np.ascontiguousarray(np.concatenate([p["order"] for p in plans]), np.uint64)
        offsets = np.ascontiguousarray(np.concatenate([p["offsets"] for p in plans]), np.uint64)
        owned = np.zeros(int(sum(int(d) for d in dims)) + 1, dtype=np.uint32)
        base = 0
        for d, p in enumerate(plans):
            owned[base:base + len(p["owned"])] = p["owned"]
            base += int(dims[d])
        owned_off = np.ascontiguousarray(np.concatenate([p["owned_offsets"] for p in plans]),
                                         np.uint64)
        totals = np.zeros(iters, dtype=np.float64)
        mode_min = np.zeros(n, dtype=np.float64)
        ident = C.c_int(0)
        f = self.lib.ref_run_timed_plans
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p, C.c_uint64,
                      np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"), _u64p, _u64p,
                      _u32p, _u64p, C.c_uint64, C.c_uint64, _f64p, _f64p, _ip]
        self._check(f(n, dims, nnz, coords, np.ascontiguousarray(values, np.float32), rank,
                      self._factor_concat(factors), kappa, schemes, orders, offsets, owned,
                      owned_off, batch_p, iters, totals, mode_min, C.byref(ident)))
        return totals, mode_min, bool(ident.value)

    def mttkrp_all_modes(self, dims, coords, values, factors, kappa, strategy=0, policy=0,
                         deterministic=True, chain=False):
        dims = _dims(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        out = np.empty(int(sum(int(d) for d in dims)) * rank, dtype=np.float32)
        f = self.lib.ref_mttkrp_all_modes
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p,
                      C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, _f32p]
        self._check(f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, np.float32),
                      rank, self._factor_concat(factors), kappa, strategy, policy,
                      int(deterministic), int(chain), out))
        mats, off = [], 0
        for d in dims:
            mats.append(out[off:off + int(d) * rank].reshape(int(d), rank))
            off += int(d) * rank
        return mats

    def run_timed(self, dims, coords, values, factors, kappa, iters, strategy=0, policy=0,
                  batch_p=32):
        """Returns (total_ms per iteration, per-mode min ms, plan build ms)."""
        dims = _dims(dims)
        rank = int(np.asarray(factors[0]).shape[1])
        coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        nnz = coords.size // len(dims)
        totals = np.zeros(iters, dtype=np.float64)
        mode_min = np.zeros(len(dims), dtype=np.float64)
        plan_ms = C.c_double(0)
        f = self.lib.ref_run_timed
        f.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f32p, C.c_uint64, _f32p,
                      C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _f64p, _f64p,
                      C.POINTER(C.c_double)]
        self._check(f(len(dims), dims, nnz, coords, np.ascontiguousarray(values, np.float32),
                      rank, self._factor_concat(factors), kappa, strategy, policy, batch_p,
                      iters, totals, mode_min, C.byref(plan_ms)))
        return totals, mode_min, plan_ms.value


def reference_available() -> bool:
    return os.path.exists(Reference.path)
