"""B200-native all-mode spMTTKRP (arxiv 2503.18198) — Python host layer.

This package mirrors the reference library's ``mttkrp`` namespace
(/root/reference/proj/core/include/mttkrp) on top of the C ABI in
``include/mttkrp_b200.h``, implemented by ``libmttkrp_b200.so`` (CUDA, sm_100a):

=====================================  ===============================================
reference (C++)                        here
=====================================  ===============================================
SparseTensorCOO<T>::from_parts         SparseTensorCOO.from_parts (tensor.hpp:45-55)
generate_synthetic                     generate_synthetic (synthetic.hpp:58-158)
random_factors                         random_factors (factor.hpp:71-84)
build_mode_plans / ModePlan            build_mode_plans / ModePlan (layout.hpp:47-149)
mode_degrees                           mode_degrees (layout.hpp:106-111)
mttkrp_mode                            mttkrp_mode (kernel.hpp:161-169)
mttkrp_all_modes                       mttkrp_all_modes (kernel.hpp:177-197)
run_timed                              run_timed (kernel.hpp:239-287)
verify_against / verify_tolerance      verify_against / verify_tolerance (verify.hpp)
parse_frostt / read_frostt_file        parse_frostt / read_frostt_file (frostt.hpp:74-199)
write_frostt(_string/_file)            write_frostt_string / write_frostt_file (:165-206)
(absent)                               save/load_tensor_cache, load_tensor (binary cache)
(absent)                   cpd_als / Context.cpd_als_iter
=====================================  ===============================================

Errors raise :class:`MttkrpError` (the reference's ``mttkrp::error``) with the
reference's message texts.  There is no CPU fallback: every compute call goes through
the CUDA library and fails loudly when it is missing or no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "MttkrpError", "Scheme", "Strategy", "SchemePolicy", "ExecConfig", "SparseTensorCOO",
    "FactorMatrix", "ModePlan", "Context", "build_mode_plans", "mttkrp_mode",
    "mttkrp_all_modes", "run_timed", "generate_synthetic", "generate_powerlaw",
    "random_factors", "verify_against", "verify_tolerance", "mode_degrees", "cpd_als",
    "element_update", "FrosttOptions", "FrosttParseResult", "parse_frostt", "read_frostt_file",
    "write_frostt_string", "write_frostt_file", "save_tensor_cache", "load_tensor_cache",
    "load_tensor",
    "load_library", "library_path", "EXPORTED_SYMBOLS",
]

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "libmttkrp_b200.so"

MK_OK, MK_EINVAL, MK_ENOMEM, MK_ECUDA, MK_ENONFINITE, MK_ESTATE, MK_ENCCL = range(7)
EXEC_FAST, EXEC_DETERMINISTIC, EXEC_PARTITIONED, EXEC_REFERENCE = 0, 1, 2, 3
PLAN_TIMED, PLAN_MODEL = 0, 1

EXPORTED_SYMBOLS = [
    "mk_last_error", "mk_version", "mk_device_count", "mk_device_sm_count", "mk_create", "mk_destroy",
    "mk_set_stream", "mk_synchronize", "mk_tensor_upload", "mk_tensor_norm2",
    "mk_build_plans", "mk_get_plan_info", "mk_fast_path_info", "mk_set_fast_kernel", "mk_set_plan_mode", "mk_plan_export", "mk_mode_degrees",
    "mk_copy_export", "mk_factors_upload", "mk_factor_upload", "mk_factor_download",
    "mk_mttkrp_mode", "mk_mttkrp_all_modes", "mk_sweep_async", "mk_mttkrp_mode_async",
    "mk_output_download",
    "mk_sweep_host", "mk_run_timed", "mk_flush_l2", "mk_last_sweep_fused", "mk_cpd_als_iter", "mk_cpd_als",
    "mk_generate_synthetic", "mk_generate_powerlaw", "mk_random_factors",
    "mk_set_shard", "mk_shard_rows", "mk_shard_pack", "mk_shard_unpack", "mk_shard_cuts",
    "mk_shard_split", "mk_shard_range", "mk_comm_unique_id", "mk_comm_init", "mk_comm_destroy",
    "mk_sweep_sharded", "mk_cpd_als_iter_sharded",
    "mk_als_update_mode", "mk_als_fit", "mk_output_device_ptr",
    "mk_tensor_upload_f64", "mk_factors_upload_f64", "mk_mttkrp_mode_f64",
    "mk_mttkrp_all_modes_f64", "mk_random_factors_f64", "mk_generate_synthetic_f64",
    "mk_frostt_parse", "mk_frostt_read_file", "mk_host_tensor_info", "mk_host_tensor_export",
    "mk_host_tensor_free", "mk_frostt_format", "mk_frostt_write_file", "mk_tensor_cache_write",
    "mk_tensor_cache_read",
]


class MttkrpError(RuntimeError):
    """mttkrp::error (types.hpp:18-21).  ``status`` is the C-ABI mk_status."""

    def __init__(self, msg: str, status: int = MK_EINVAL):
        super().__init__(msg)
        self.status = status


class Scheme(enum.IntEnum):  # layout.hpp:17
    scheme1 = 1
    scheme2 = 2


class Strategy(enum.IntEnum):  # layout.hpp:22
    cyclic = 0
    least_loaded = 1


class SchemePolicy(enum.IntEnum):  # layout.hpp:24
    adaptive = 0
    scheme1_only = 1
    scheme2_only = 2


class _PlanInfo(C.Structure):
    _fields_ = [("scheme", C.c_int), ("kappa", C.c_uint64), ("nnz", C.c_uint64),
                ("owned_total", C.c_uint64), ("distinct_rows", C.c_uint64),
                ("split_rows", C.c_uint64), ("device_bytes", C.c_uint64)]


class _FastInfo(C.Structure):
    """mk_fast_info: the fast path's kernel choice and plan for one mode copy."""
    _fields_ = [("kernel", C.c_int), ("blocked", C.c_int), ("blocks", C.c_uint32),
                ("staged_levels", C.c_uint32), ("outer_level", C.c_int),
                ("launches", C.c_uint32), ("stream_bytes", C.c_uint64)]

    KERNELS = {-1: "undecided", 0: "k_stream2 (level-ordered)", 1: "k_mttkrp_stream (fiber-ordered)",
               2: "k_mttkrp_tiles"}

    def as_dict(self):
        return {"kernel": self.KERNELS.get(self.kernel, str(self.kernel)), "blocked": bool(self.blocked),
                "blocks": int(self.blocks), "staged_levels": int(self.staged_levels),
                "outer_level": bool(self.outer_level), "launches": int(self.launches),
                "stream_bytes": int(self.stream_bytes)}


_lib_lock = threading.Lock()
_lib_handle: Optional[C.CDLL] = None


def library_path() -> str:
    # MKB_LIB: an alternative build of the same library (kernel-variant experiments)
    return os.environ.get("MKB_LIB") or os.path.join(HERE, _LIB_NAME)


def load_library() -> C.CDLL:
    """Load libmttkrp_b200.so (raises if it was not built — no fallback)."""
    global _lib_handle
    with _lib_lock:
        if _lib_handle is not None:
            return _lib_handle
        path = library_path()
        if not os.path.exists(path):
            raise MttkrpError(f"CUDA extension not built: {path} (run __graft_entry__.build())",
                              MK_ESTATE)
        lib = C.CDLL(path)
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        P = C.POINTER
        sig = {
            "mk_last_error": (C.c_char_p, []),
            "mk_version": (C.c_char_p, []),
            "mk_device_count": (i32, [P(i32)]),
            "mk_device_sm_count": (i32, [i32, P(i32)]),
            "mk_create": (i32, [i32, P(vp)]),
            "mk_destroy": (i32, [vp]),
            "mk_set_stream": (i32, [vp, vp]),
            "mk_synchronize": (i32, [vp]),
            "mk_tensor_upload": (i32, [vp, u32, vp, u64, vp, vp]),
            "mk_tensor_norm2": (i32, [vp, P(C.c_double)]),
            "mk_build_plans": (i32, [vp, u64, i32, i32]),
            "mk_get_plan_info": (i32, [vp, u32, P(_PlanInfo)]),
            "mk_fast_path_info": (i32, [vp, u32, P(_FastInfo)]),
            "mk_set_fast_kernel": (i32, [vp, i32]),
            "mk_set_plan_mode": (i32, [vp, i32]),
            "mk_plan_export": (i32, [vp, u32, vp, vp, vp, vp]),
            "mk_mode_degrees": (i32, [vp, u32, vp]),
            "mk_copy_export": (i32, [vp, u32, vp, vp]),
            "mk_factors_upload": (i32, [vp, u32, vp]),
            "mk_factor_upload": (i32, [vp, u32, vp]),
            "mk_factor_download": (i32, [vp, u32, vp]),
            "mk_mttkrp_mode": (i32, [vp, u32, i32, vp]),
            "mk_mttkrp_all_modes": (i32, [vp, i32, i32, vp]),
            "mk_sweep_async": (i32, [vp, i32, i32]),
            "mk_mttkrp_mode_async": (i32, [vp, u32, i32]),
            "mk_output_download": (i32, [vp, u32, vp]),
            "mk_sweep_host": (i32, [vp, vp, vp, i32, i32]),
            "mk_run_timed": (i32, [vp, u64, i32, i32, vp, vp, P(i32)]),
            "mk_flush_l2": (i32, [vp]),
            "mk_last_sweep_fused": (i32, [vp, P(C.c_int)]),
            "mk_cpd_als_iter": (i32, [vp, P(C.c_double), vp]),
            "mk_cpd_als": (i32, [vp, u64, C.c_double, P(C.c_double), P(u64), vp]),
            "mk_generate_synthetic": (i32, [u32, vp, u64, i32, u64, u64, u64, vp, vp]),
            "mk_generate_powerlaw": (i32, [u32, vp, u64, C.c_double, u64, vp, vp]),
            "mk_random_factors": (i32, [u32, vp, u64, u64, vp]),
            "mk_set_shard": (i32, [vp, u32, u32]),
            "mk_shard_rows": (i32, [vp, u32, u32, P(u64), P(u64)]),
            "mk_shard_pack": (i32, [vp, u32, vp]),
            "mk_shard_unpack": (i32, [vp, u32, vp, u64]),
            "mk_shard_cuts": (i32, [vp, u64, u32, vp]),
            "mk_shard_split": (i32, [vp, u64, u32, vp]),
            "mk_comm_unique_id": (i32, [vp]),
            "mk_comm_init": (i32, [vp, u32, u32, vp]),
            "mk_comm_destroy": (i32, [vp]),
            "mk_sweep_sharded": (i32, [vp]),
            "mk_cpd_als_iter_sharded": (i32, [vp, P(C.c_double), vp]),
            "mk_shard_range": (i32, [vp, u32, u32, P(u64), P(u64), P(u64), P(u64)]),
            "mk_als_update_mode": (i32, [vp, u32]),
            "mk_als_fit": (i32, [vp, P(C.c_double), vp]),
            "mk_output_device_ptr": (i32, [vp, u32, P(vp)]),
            "mk_tensor_upload_f64": (i32, [vp, u32, vp, u64, vp, vp]),
            "mk_factors_upload_f64": (i32, [vp, u32, vp]),
            "mk_mttkrp_mode_f64": (i32, [vp, u32, i32, vp]),
            "mk_mttkrp_all_modes_f64": (i32, [vp, i32, i32, vp]),
            "mk_random_factors_f64": (i32, [u32, vp, u64, u64, vp]),
            "mk_generate_synthetic_f64": (i32, [u32, vp, u64, i32, u64, u64, u64, vp, vp]),
            "mk_frostt_parse": (i32, [C.c_char_p, u64, i32, i32, vp, u32, u32, P(vp)]),
            "mk_frostt_read_file": (i32, [C.c_char_p, i32, i32, vp, u32, u32, P(vp)]),
            "mk_host_tensor_info": (i32, [vp, P(u32), vp, u32, P(u64), P(u64), P(i32)]),
            "mk_host_tensor_export": (i32, [vp, vp, vp]),
            "mk_host_tensor_free": (i32, [vp]),
            "mk_frostt_format": (i32, [u32, u64, vp, vp, i32, u32, vp, u64, P(u64)]),
            "mk_frostt_write_file": (i32, [C.c_char_p, u32, u64, vp, vp, i32, u32]),
            "mk_tensor_cache_write": (i32, [C.c_char_p, u32, vp, u64, vp, vp, i32]),
            "mk_tensor_cache_read": (i32, [C.c_char_p, P(vp)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib_handle = lib
        return lib


def _check(rc: int) -> None:
    if rc != MK_OK:
        msg = load_library().mk_last_error().decode()
        raise MttkrpError(msg, rc)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _ptr_array(arrs: Sequence[np.ndarray]):
    return (C.c_void_p * len(arrs))(*[_ptr(a) for a in arrs])


# ----------------------------------------------------------------------------- data model
class SparseTensorCOO:
    """COO tensor (tensor.hpp:34-111): shape + nnz×N uint32 coordinates + fp32 values."""

    def __init__(self, dims: Sequence[int], coords=None, values=None, validate: bool = True):
        dims = [int(d) for d in dims]
        if not dims:
            raise MttkrpError("shape: a tensor needs at least one mode")
        if any(d <= 0 for d in dims):
            raise MttkrpError("shape: zero extent")
        if any(d > 0xFFFFFFFF for d in dims):
            raise MttkrpError("shape: extent exceeds 2^32-1")
        self.dims = dims
        n = len(dims)
        if coords is None:
            coords = np.zeros((0, n), dtype=np.uint32)
            values = np.zeros(0, dtype=np.float32)
        coords = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(-1, n)
                                      if not (isinstance(coords, np.ndarray)
                                              and coords.dtype == np.uint32)
                                      else coords.reshape(-1, n))
        vdt = np.float64 if (isinstance(values, np.ndarray) and values.dtype == np.float64) \
            else np.float32  # SparseTensorCOO<double> when given fp64 values
        values = np.ascontiguousarray(np.asarray(values, dtype=vdt).reshape(-1))
        if coords.shape[0] != values.shape[0]:
            raise MttkrpError("tensor: coordinate/value storage size mismatch")
        if validate:
            self._validate(coords, values)
        self.coords = np.ascontiguousarray(coords.astype(np.uint32, copy=False))
        self.values = values
        self._ctx: Optional["Context"] = None

    from_parts = classmethod(lambda cls, dims, coords, values: cls(dims, coords, values))

    def _validate(self, coords, values):  # tensor.hpp:97-106, first bad element first
        if coords.size == 0:
            return
        dims = np.asarray(self.dims, dtype=np.int64)
        c64 = coords.astype(np.int64, copy=False)
        bad_c = (c64 < 0) | (c64 >= dims[None, :])
        bad_row_c = bad_c.any(axis=1)
        bad_v = ~np.isfinite(values)
        first_c = int(np.argmax(bad_row_c)) if bad_row_c.any() else None
        first_v = int(np.argmax(bad_v)) if bad_v.any() else None
        if first_c is not None and (first_v is None or first_c <= first_v):
            h = int(np.argmax(bad_c[first_c]))
            raise MttkrpError(f"tensor: coordinate {int(c64[first_c, h])} out of range for mode {h}")
        if first_v is not None:
            raise MttkrpError("tensor: non-finite element value")

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def mode_count(self) -> int:
        return len(self.dims)

    def extent(self, d: int) -> int:
        return self.dims[d]

    def index(self, i: int, mode: int) -> int:
        return int(self.coords[i, mode])


@dataclass
class FactorMatrix:
    """Dense row-major I_d × R factor (factor.hpp:16-48)."""
    mode: int
    data: np.ndarray  # float32 (rows, rank)

    def __post_init__(self):
        dt = np.float64 if (isinstance(self.data, np.ndarray) and self.data.dtype == np.float64) \
            else np.float32  # FactorMatrix<double> stays fp64
        self.data = np.ascontiguousarray(np.asarray(self.data, dtype=dt))
        if self.data.ndim != 2:
            raise MttkrpError("factor: matrix must be 2-D")

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    @property
    def rank(self) -> int:
        return int(self.data.shape[1])

    @staticmethod
    def zeros(mode: int, rows: int, rank: int) -> "FactorMatrix":
        return FactorMatrix(mode, np.zeros((rows, rank), dtype=np.float32))

    def at(self, i: int, r: int) -> float:
        return float(self.data[i, r])


@dataclass
class ExecConfig:
    """kernel.hpp:23-34.  kappa must match the plans; batch_p is accepted for API parity
    (it has no semantic effect in the reference either, kernel.hpp:95-97)."""
    kappa: int = 1
    batch_p: int = 32
    deterministic: bool = False
    # the reference's work split on the GPU (partition z of the plan on CTA z; the paper's
    # scheme ablation, MK_EXEC_PARTITIONED); no reference counterpart flag
    partitioned: bool = False
    # the reference's parallel-executor contract (MK_EXEC_REFERENCE: Scheme 1 modes bitwise
    # equal to deterministic) -- the C++ drop-in's default.  This harness
    # API defaults to the B200 fast path (MK_EXEC_FAST, within 1e-4 of the oracle).
    reference: bool = False

    def exec_code(self) -> int:
        if self.deterministic:
            return EXEC_DETERMINISTIC
        if self.partitioned:
            return EXEC_PARTITIONED
        return EXEC_REFERENCE if self.reference else EXEC_FAST

    def validate(self):
        if self.kappa < 1:
            raise MttkrpError("kernel: kappa must be at least 1")
        if self.batch_p < 1:
            raise MttkrpError("kernel: batch size P must be at least 1")


# ----------------------------------------------------------------------------- device context
class Context:
    """One mk_context: device-resident tensor, mode copies, factors and outputs."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        _check(self.lib.mk_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.dims: List[int] = []
        self.nnz = 0
        self.rank = 0
        self.kappa = 0
        self._factor_key = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.mk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: Optional[int]):
        """Enqueue on the given cudaStream_t (0 = CUDA legacy default stream, None = the
        context's own stream)."""
        handle = C.c_void_p(-1) if stream_ptr is None else C.c_void_p(stream_ptr)
        _check(self.lib.mk_set_stream(self.h, handle))

    def synchronize(self):
        _check(self.lib.mk_synchronize(self.h))

    # tensor / plans
    def upload_tensor(self, t: SparseTensorCOO):
        dims = np.asarray(t.dims, dtype=np.uint32)
        up = self.lib.mk_tensor_upload_f64 if t.values.dtype == np.float64 else \
            self.lib.mk_tensor_upload
        _check(up(self.h, len(t.dims), _ptr(dims), t.nnz, _ptr(t.coords), _ptr(t.values)))
        self.f64 = t.values.dtype == np.float64
        self.rank64 = 0
        self.dims = list(t.dims)
        self.nnz = t.nnz
        self.rank = 0
        self._factor_key = None

    def norm2(self) -> float:
        v = C.c_double()
        _check(self.lib.mk_tensor_norm2(self.h, C.byref(v)))
        return v.value

    def build_plans(self, kappa: int, strategy=Strategy.cyclic, policy=SchemePolicy.adaptive):
        if kappa < 1:
            raise MttkrpError("layout: kappa must be at least 1")
        _check(self.lib.mk_build_plans(self.h, int(kappa), int(strategy), int(policy)))
        self.kappa = int(kappa)

    def plan_info(self, mode: int) -> _PlanInfo:
        info = _PlanInfo()
        _check(self.lib.mk_get_plan_info(self.h, mode, C.byref(info)))
        return info

    def fast_path_info(self, mode: int) -> _FastInfo:
        info = _FastInfo()
        _check(self.lib.mk_fast_path_info(self.h, mode, C.byref(info)))
        return info

    def set_fast_kernel(self, kernel: int):
        """Force the fast path's kernel (0 level-ordered, 1 fiber-ordered, 2 tiles; -1 = timed choice)."""
        _check(self.lib.mk_set_fast_kernel(self.h, int(kernel)))

    def set_plan_mode(self, mode: int):
        """PLAN_TIMED (0, default): time the candidate plans on the first fast call of a mode;
        PLAN_MODEL (1): the cost model's plan, no timing (reproducible across runs and boxes)."""
        _check(self.lib.mk_set_plan_mode(self.h, int(mode)))

    def plan_export(self, mode: int):
        info = self.plan_info(mode)
        order = np.empty(max(self.nnz, 1), dtype=np.uint64)
        offs = np.empty(info.kappa + 1, dtype=np.uint64)
        owned = np.empty(max(info.owned_total, 1), dtype=np.uint32)
        owned_off = np.empty(info.kappa + 1, dtype=np.uint64)
        _check(self.lib.mk_plan_export(self.h, mode, _ptr(order), _ptr(offs), _ptr(owned),
                                       _ptr(owned_off)))
        return {"scheme": info.scheme, "order": order[:self.nnz], "offsets": offs,
                "owned": owned[:info.owned_total], "owned_offsets": owned_off}

    def copy_export(self, mode: int):
        n = len(self.dims)
        idx = np.empty((n, max(self.nnz, 1)), dtype=np.uint32)
        vals = np.empty(max(self.nnz, 1), dtype=np.float32)
        _check(self.lib.mk_copy_export(self.h, mode, _ptr(idx), _ptr(vals)))
        return idx[:, :self.nnz], vals[:self.nnz]

    def mode_degrees(self, mode: int) -> np.ndarray:
        out = np.empty(self.dims[mode], dtype=np.uint64)
        _check(self.lib.mk_mode_degrees(self.h, mode, _ptr(out)))
        return out

    # factors
    def upload_factors(self, factors: Sequence[np.ndarray]):
        mats = [np.ascontiguousarray(np.asarray(f, dtype=np.float32)) for f in factors]
        rank = int(mats[0].shape[1])
        _check(self.lib.mk_factors_upload(self.h, rank, _ptr_array(mats)))
        self.rank = rank

    def upload_factors_f64(self, factors: Sequence[np.ndarray]):
        """FactorMatrix<double> inputs of the fp64 path."""
        mats = [np.ascontiguousarray(np.asarray(f, dtype=np.float64)) for f in factors]
        rank = int(mats[0].shape[1])
        _check(self.lib.mk_factors_upload_f64(self.h, rank, _ptr_array(mats)))
        self.rank64 = rank

    def mttkrp_mode_f64(self, mode: int, deterministic: bool = False) -> np.ndarray:
        out = np.empty((self.dims[mode], self.rank64), dtype=np.float64)
        _check(self.lib.mk_mttkrp_mode_f64(self.h, mode, int(deterministic), _ptr(out)))
        return out

    def mttkrp_all_modes_f64(self, chain: bool = False, deterministic: bool = False):
        outs = [np.empty((d, self.rank64), dtype=np.float64) for d in self.dims]
        _check(self.lib.mk_mttkrp_all_modes_f64(self.h, int(chain), int(deterministic),
                                                _ptr_array(outs)))
        return outs

    def download_factor(self, mode: int) -> np.ndarray:
        out = np.empty((self.dims[mode], self.rank), dtype=np.float32)
        _check(self.lib.mk_factor_download(self.h, mode, _ptr(out)))
        return out

    # compute
    def mttkrp_mode(self, mode: int, deterministic: bool = False) -> np.ndarray:
        out = np.empty((self.dims[mode], self.rank), dtype=np.float32)
        _check(self.lib.mk_mttkrp_mode(self.h, mode, int(deterministic), _ptr(out)))
        return out

    def mttkrp_all_modes(self, chain: bool = False, deterministic: bool = False):
        outs = [np.empty((d, self.rank), dtype=np.float32) for d in self.dims]
        _check(self.lib.mk_mttkrp_all_modes(self.h, int(chain), int(deterministic),
                                            _ptr_array(outs)))
        return outs

    def sweep_async(self, chain: bool = False, deterministic: bool = False):
        _check(self.lib.mk_sweep_async(self.h, int(chain), int(deterministic)))

    def mttkrp_mode_async(self, mode: int, deterministic: bool = False):
        _check(self.lib.mk_mttkrp_mode_async(self.h, mode, int(deterministic)))

    def output(self, mode: int) -> np.ndarray:
        out = np.empty((self.dims[mode], self.rank), dtype=np.float32)
        _check(self.lib.mk_output_download(self.h, mode, _ptr(out)))
        return out

    def sweep_host(self, factors_host: Sequence[np.ndarray], outs_host: Sequence[np.ndarray],
                   chain: bool = False, deterministic: bool = False):
        _check(self.lib.mk_sweep_host(self.h, _ptr_array(factors_host), _ptr_array(outs_host),
                                      int(chain), int(deterministic)))

    def run_timed(self, iters: int, deterministic: bool = False, flush_l2: bool = True):
        n = len(self.dims)
        mode_ms = np.zeros((iters, n), dtype=np.float64)
        total = np.zeros(iters, dtype=np.float64)
        same = C.c_int(0)
        _check(self.lib.mk_run_timed(self.h, iters, int(deterministic), int(flush_l2),
                                     _ptr(mode_ms), _ptr(total), C.byref(same)))
        self.last_outputs_bit_identical = bool(same.value)
        return mode_ms, total

    def flush_l2(self):
        _check(self.lib.mk_flush_l2(self.h))

    def last_sweep_fused(self) -> bool:
        """Whether the last all-mode sweep ran as one fused launch (k_sweep2)."""
        v = C.c_int(0)
        _check(self.lib.mk_last_sweep_fused(self.h, C.byref(v)))
        return bool(v.value)

    # multi-GPU shards
    def set_shard(self, rank: int, world: int):
        _check(self.lib.mk_set_shard(self.h, rank, world))

    def shard_rows(self, mode: int, rank: int):
        k0, k1 = C.c_uint64(), C.c_uint64()
        _check(self.lib.mk_shard_rows(self.h, mode, rank, C.byref(k0), C.byref(k1)))
        return int(k0.value), int(k1.value)

    # ---- NCCL inside the library (comm.cu)
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(load_library().mk_comm_unique_id(buf))
        return buf.raw

    def comm_init(self, world: int, rank: int, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(self.lib.mk_comm_init(self.h, world, rank, buf))

    def comm_destroy(self):
        _check(self.lib.mk_comm_destroy(self.h))

    def sweep_sharded(self):
        _check(self.lib.mk_sweep_sharded(self.h))

    def cpd_als_iter_sharded(self):
        fit = C.c_double()
        lam = np.empty(max(self.rank, 1), dtype=np.float32)
        _check(self.lib.mk_cpd_als_iter_sharded(self.h, C.byref(fit), _ptr(lam)))
        return fit.value, lam

    def shard_range(self, mode: int, rank: int):
        """(e0, e1, k0, k1): owned elements and touched copy rows of `rank` in `mode`."""
        v = [C.c_uint64() for _ in range(4)]
        _check(self.lib.mk_shard_range(self.h, mode, rank, *[C.byref(x) for x in v]))
        return tuple(int(x.value) for x in v)

    def shard_pack(self, mode: int, dst):
        """dst: device pointer or CUDA tensor (>= owned rows x R fp32)."""
        ptr = dst.data_ptr() if hasattr(dst, "data_ptr") else int(dst)
        _check(self.lib.mk_shard_pack(self.h, mode, C.c_void_p(ptr)))

    def shard_unpack(self, mode: int, src, stride_rows: int):
        """src: device pointer or CUDA tensor (world x stride_rows x R fp32)."""
        ptr = src.data_ptr() if hasattr(src, "data_ptr") else int(src)
        _check(self.lib.mk_shard_unpack(self.h, mode, C.c_void_p(ptr), stride_rows))

    def output_device_ptr(self, mode: int) -> int:
        p = C.c_void_p()
        _check(self.lib.mk_output_device_ptr(self.h, mode, C.byref(p)))
        return int(p.value or 0)

    def als_update_mode(self, mode: int):
        _check(self.lib.mk_als_update_mode(self.h, mode))

    def als_fit(self):
        fit = C.c_double()
        lam = np.empty(self.rank, dtype=np.float32)
        _check(self.lib.mk_als_fit(self.h, C.byref(fit), _ptr(lam)))
        return fit.value, lam

    def cpd_als_iter(self):
        fit = C.c_double()
        lam = np.empty(self.rank, dtype=np.float32)
        _check(self.lib.mk_cpd_als_iter(self.h, C.byref(fit), _ptr(lam)))
        return fit.value, lam

    def cpd_als(self, max_iters: int, tol: float = 1e-5):
        fit = C.c_double()
        done = C.c_uint64()
        lam = np.empty(self.rank, dtype=np.float32)
        _check(self.lib.mk_cpd_als(self.h, max_iters, tol, C.byref(fit), C.byref(done), _ptr(lam)))
        return fit.value, int(done.value), lam


# ----------------------------------------------------------------------------- plans
class ModePlan:
    """layout.hpp:47-64.  The copy lives on the device; order / offsets / owned indices
    are exported on first access (bit-exact with the reference's ModePlan)."""

    def __init__(self, ctx: Context, mode: int, tensor: SparseTensorCOO):
        self._ctx = ctx
        self._tensor = tensor
        self.mode = mode
        info = ctx.plan_info(mode)
        self.scheme = Scheme(info.scheme)
        self.kappa = int(info.kappa)
        self._nnz = int(info.nnz)
        self._export = None

    def _ex(self):
        if self._export is None:
            self._export = self._ctx.plan_export(self.mode)
        return self._export

    @property
    def order(self) -> np.ndarray:
        return self._ex()["order"]

    @property
    def partition_offsets(self) -> np.ndarray:
        return self._ex()["offsets"]

    @property
    def owned_indices(self) -> List[np.ndarray]:
        ex = self._ex()
        if self.scheme != Scheme.scheme1:
            return []
        o, off = ex["owned"], ex["owned_offsets"]
        return [o[int(off[z]):int(off[z + 1])] for z in range(self.kappa)]

    def nnz(self) -> int:
        return self._nnz

    def partition_size(self, z: int) -> int:
        off = self.partition_offsets
        return int(off[z + 1] - off[z])


def _context_for(t: SparseTensorCOO) -> Context:
    if t._ctx is None:
        t._ctx = Context()
        t._ctx.upload_tensor(t)
    return t._ctx


def build_mode_plans(t: SparseTensorCOO, kappa: int, strategy=Strategy.cyclic,
                     policy=SchemePolicy.adaptive) -> List[ModePlan]:
    """layout.hpp:131-149 — all N mode copies built on the device.  Every call owns a new
    device session (as the C++ header's Session), so plans of an earlier call (another kappa
    or policy on the same tensor) keep describing — and running on — their own copies."""
    if kappa < 1:
        raise MttkrpError("layout: kappa must be at least 1")
    ctx = Context()
    ctx.upload_tensor(t)
    ctx.build_plans(kappa, strategy, policy)
    t._ctx = ctx  # the latest session also serves mode_degrees
    return [ModePlan(ctx, d, t) for d in range(t.mode_count())]


def mode_degrees(t: SparseTensorCOO, d: int) -> np.ndarray:
    """layout.hpp:106-111 (needs plans built for the tensor)."""
    if d >= t.mode_count():
        raise MttkrpError("layout: mode out of range")
    return _context_for(t).mode_degrees(d)


# ----------------------------------------------------------------------------- kernels
def _validate_factors(t: SparseTensorCOO, factors: Sequence[FactorMatrix]):  # kernel.hpp:44-61
    if len(factors) != t.mode_count():
        raise MttkrpError("kernel: expected one factor matrix per mode")
    rank = factors[0].rank if factors else 0
    if rank < 1:
        raise MttkrpError("kernel: rank must be at least 1")
    for w, f in enumerate(factors):
        if f.mode != w:
            raise MttkrpError(f"kernel: factor matrix {w} labeled mode {f.mode}")
        if f.rows != t.extent(w):
            raise MttkrpError(f"kernel: factor matrix {w} has {f.rows} rows, tensor extent is "
                              f"{t.extent(w)}")
        if f.rank != rank:
            raise MttkrpError("kernel: factor matrices disagree on rank")


def _validate_plan(t: SparseTensorCOO, plan: ModePlan, config: ExecConfig):  # kernel.hpp:63-73
    if plan.mode >= t.mode_count():
        raise MttkrpError("kernel: plan mode out of range")
    if plan._tensor is not t or plan.nnz() != t.nnz:
        raise MttkrpError("kernel: plan does not cover this tensor")
    off = plan.partition_offsets
    if len(off) != plan.kappa + 1 or int(off[0]) != 0 or int(off[-1]) != t.nnz:
        raise MttkrpError("kernel: malformed partition offsets")
    if plan.kappa != config.kappa:
        raise MttkrpError(f"kernel: plan built for kappa {plan.kappa}, config requests "
                          f"{config.kappa}")


def _as_factors(factors) -> List[FactorMatrix]:
    return [f if isinstance(f, FactorMatrix) else FactorMatrix(i, f) for i, f in enumerate(factors)]


def _is_f64(t: SparseTensorCOO, factors: Sequence[FactorMatrix]) -> bool:
    """T = double: an fp64 tensor takes fp64 factors (the reference's templates do not mix T)."""
    f64 = [f.data.dtype == np.float64 for f in factors]
    if t.values.dtype == np.float64 and not all(f64):
        raise MttkrpError("kernel: an fp64 tensor needs fp64 factor matrices")
    if t.values.dtype != np.float64 and any(f64):
        raise MttkrpError("kernel: fp64 factor matrices need an fp64 tensor")
    return t.values.dtype == np.float64


def _upload_if_changed(ctx: Context, factors: Sequence[FactorMatrix]):
    ctx.upload_factors([f.data for f in factors])


def mttkrp_mode(t: SparseTensorCOO, plan: ModePlan, factors, config: ExecConfig) -> FactorMatrix:
    """kernel.hpp:161-169 on the device."""
    factors = _as_factors(factors)
    config.validate()
    _validate_factors(t, factors)
    _validate_plan(t, plan, config)
    ctx = plan._ctx
    if _is_f64(t, factors):
        ctx.upload_factors_f64([f.data for f in factors])
        return FactorMatrix(plan.mode, ctx.mttkrp_mode_f64(plan.mode, config.deterministic))
    _upload_if_changed(ctx, factors)
    return FactorMatrix(plan.mode, ctx.mttkrp_mode(plan.mode, config.exec_code()))


def mttkrp_all_modes(t: SparseTensorCOO, plans: Sequence[ModePlan], factors, config: ExecConfig,
                     chain_outputs: bool) -> List[FactorMatrix]:
    """kernel.hpp:177-197 on the device (stream order = the global barrier)."""
    factors = _as_factors(factors)
    if len(plans) != t.mode_count():
        raise MttkrpError("kernel: expected one plan per mode")
    for d, p in enumerate(plans):
        if p.mode != d:
            raise MttkrpError("kernel: plans out of mode order")
    config.validate()
    _validate_factors(t, factors)
    for p in plans:
        _validate_plan(t, p, config)
    ctx = plans[0]._ctx
    if _is_f64(t, factors):
        ctx.upload_factors_f64([f.data for f in factors])
        outs = ctx.mttkrp_all_modes_f64(chain_outputs, config.deterministic)
        return [FactorMatrix(d, o) for d, o in enumerate(outs)]
    _upload_if_changed(ctx, factors)
    outs = ctx.mttkrp_all_modes(chain_outputs, config.exec_code())
    return [FactorMatrix(d, o) for d, o in enumerate(outs)]


def element_update(t: SparseTensorCOO, element: int, factors, output_mode: int) -> np.ndarray:
    """kernel.hpp:133-153 (host arithmetic, API parity): acc[r] = value * prod_{w != d}
    Y_w(c_w, r), multiplied in ascending mode order."""
    factors = _as_factors(factors)
    rank = factors[0].rank if factors else 0
    if any(f.rank != rank for f in factors):
        raise MttkrpError("kernel: factor matrices disagree on rank")
    dt = t.values.dtype
    acc = np.full(rank, t.values[element], dtype=dt)
    for w, f in enumerate(factors):
        if w != output_mode:
            acc = (acc * f.data[int(t.coords[element, w])].astype(dt)).astype(dt)
    return acc


@dataclass
class ModeTiming:  # kernel.hpp:199-207
    mode: int
    scheme: Scheme
    wall_ms: List[float]
    min_ms: float
    median_ms: float
    busy_workers: int
    elements_per_worker: List[int]


@dataclass
class TimingReport:  # kernel.hpp:209-218
    iters: int
    modes: List[ModeTiming]
    total_ms: List[float]
    total_min_ms: float
    total_median_ms: float
    outputs_bit_identical: bool = True


def run_timed(t: SparseTensorCOO, plans: Sequence[ModePlan], factors, config: ExecConfig,
              iters: int, flush_l2: bool = True):
    """kernel.hpp:239-287: per-mode times from CUDA events (the reference uses
    steady_clock around each host call).  Returns (TimingReport, outputs)."""
    if iters < 1:
        raise MttkrpError("kernel: iters must be at least 1")
    factors = _as_factors(factors)
    config.validate()
    _validate_factors(t, factors)
    for p in plans:
        _validate_plan(t, p, config)
    ctx = plans[0]._ctx
    _upload_if_changed(ctx, factors)
    mode_ms, total = ctx.run_timed(iters, config.exec_code(), flush_l2)
    modes = []
    for d, p in enumerate(plans):
        sizes = [p.partition_size(z) for z in range(p.kappa)]
        w = [float(x) for x in mode_ms[:, d]]
        modes.append(ModeTiming(d, p.scheme, w, min(w), float(np.median(w)),
                                sum(1 for s in sizes if s > 0), sizes))
    report = TimingReport(iters, modes, [float(x) for x in total], float(total.min()),
                          float(np.median(total)), ctx.last_outputs_bit_identical)
    outs = [FactorMatrix(d, ctx.output(d)) for d in range(t.mode_count())]
    return report, outs


def cpd_als(t: SparseTensorCOO, plans: Sequence[ModePlan], factors, max_iters: int,
            tol: float = 1e-5):
    """CPD-ALS driver on the device (no reference counterpart)."""
    factors = _as_factors(factors)
    _validate_factors(t, factors)
    ctx = plans[0]._ctx
    ctx.upload_factors([f.data for f in factors])
    fit, iters, lam = ctx.cpd_als(max_iters, tol)
    out = [FactorMatrix(d, ctx.download_factor(d)) for d in range(t.mode_count())]
    return fit, iters, lam, out


# ----------------------------------------------------------------------------- ingest (host)
def generate_synthetic(dims, nnz, dist="uniform", skew_mode=0, skew_distinct=2,
                       seed=0, dtype=np.float32) -> SparseTensorCOO:
    """synthetic.hpp:58-158, bit-identical (host C++ in libmttkrp_b200.so); dtype=np.float64
    gives generate_synthetic<double>."""
    lib = load_library()
    d = np.asarray(dims, dtype=np.uint32)
    coords = np.empty((nnz, len(dims)), dtype=np.uint32)
    f64 = np.dtype(dtype) == np.float64
    vals = np.empty(nnz, dtype=np.float64 if f64 else np.float32)
    dist_i = {"uniform": 0, "mode_skewed": 1}[dist] if isinstance(dist, str) else int(dist)
    gen = lib.mk_generate_synthetic_f64 if f64 else lib.mk_generate_synthetic
    _check(gen(len(dims), _ptr(d), nnz, dist_i, skew_mode, skew_distinct, seed, _ptr(coords),
               _ptr(vals)))
    return SparseTensorCOO(dims, coords, vals, validate=False)


def generate_powerlaw(dims, nnz, exponent=1.0, seed=0) -> SparseTensorCOO:
    """DESIGN.md §5 power-law generator (nips-shaped config)."""
    lib = load_library()
    d = np.asarray(dims, dtype=np.uint32)
    coords = np.empty((nnz, len(dims)), dtype=np.uint32)
    vals = np.empty(nnz, dtype=np.float32)
    _check(lib.mk_generate_powerlaw(len(dims), _ptr(d), nnz, float(exponent), seed,
                                    _ptr(coords), _ptr(vals)))
    return SparseTensorCOO(dims, coords, vals, validate=False)


def random_factors(dims, rank, seed, dtype=np.float32) -> List[FactorMatrix]:
    """factor.hpp:71-84, bit-identical (T = float, or T = double with dtype=np.float64)."""
    lib = load_library()
    if rank < 1:
        raise MttkrpError("factor: rank must be at least 1")
    d = np.asarray(dims, dtype=np.uint32)
    f64 = np.dtype(dtype) == np.float64
    mats = [np.empty((int(x), rank), dtype=np.float64 if f64 else np.float32) for x in dims]
    gen = lib.mk_random_factors_f64 if f64 else lib.mk_random_factors
    _check(gen(len(dims), _ptr(d), rank, seed, _ptr_array(mats)))
    return [FactorMatrix(i, m) for i, m in enumerate(mats)]


@dataclass
class FrosttOptions:  # frostt.hpp:22-29
    merge_duplicates: bool = True
    dims_override: Optional[Sequence[int]] = None


@dataclass
class FrosttParseResult:  # frostt.hpp:31-35
    tensor: SparseTensorCOO
    duplicates_merged: int = 0


def _prec_of(dtype) -> int:
    return 64 if np.dtype(dtype) == np.float64 else 32


def _take_host_tensor(handle) -> Tuple[SparseTensorCOO, int]:
    lib = load_library()
    try:
        n, nnz, dups, prec = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_int()
        dims = np.zeros(64, dtype=np.uint32)
        _check(lib.mk_host_tensor_info(handle, C.byref(n), _ptr(dims), 64, C.byref(nnz),
                                       C.byref(dups), C.byref(prec)))
        coords = np.empty((nnz.value, n.value), dtype=np.uint32)
        vals = np.empty(nnz.value, dtype=np.float64 if prec.value == 64 else np.float32)
        _check(lib.mk_host_tensor_export(handle, _ptr(coords), _ptr(vals)))
    finally:
        lib.mk_host_tensor_free(handle)
    # the parser already validated bounds (inferred or checked extents) and finiteness
    return SparseTensorCOO([int(x) for x in dims[:n.value]], coords, vals,
                           validate=False), int(dups.value)


def _override_args(opt: Optional[FrosttOptions]):
    ovr = None if opt is None or not opt.dims_override else \
        np.asarray(opt.dims_override, dtype=np.uint32)
    merge = 1 if opt is None or opt.merge_duplicates else 0
    return merge, (None if ovr is None else _ptr(ovr)), (0 if ovr is None else ovr.size), ovr


def parse_frostt(text, options: Optional[FrosttOptions] = None, dtype=np.float32,
                 threads: int = 0) -> FrosttParseResult:
    """frostt.hpp:74-160 parse_frostt<T> on a string (multithreaded host C++)."""
    lib = load_library()
    raw = text.encode() if isinstance(text, str) else bytes(text)
    merge, op, on, _keep = _override_args(options)
    h = C.c_void_p()
    _check(lib.mk_frostt_parse(raw, len(raw), _prec_of(dtype), merge, op, on, threads,
                               C.byref(h)))
    t, dups = _take_host_tensor(h)
    return FrosttParseResult(t, dups)


def read_frostt_file(path, options: Optional[FrosttOptions] = None, dtype=np.float32,
                     threads: int = 0) -> FrosttParseResult:
    """frostt.hpp:194-199 read_frostt_file<T>."""
    lib = load_library()
    merge, op, on, _keep = _override_args(options)
    h = C.c_void_p()
    _check(lib.mk_frostt_read_file(os.fsencode(path), _prec_of(dtype), merge, op, on, threads,
                                   C.byref(h)))
    t, dups = _take_host_tensor(h)
    return FrosttParseResult(t, dups)


def _value_prec(t: SparseTensorCOO) -> int:
    return 64 if t.values.dtype == np.float64 else 32


def write_frostt_string(t: SparseTensorCOO, threads: int = 0) -> str:
    """frostt.hpp:165-192 write_frostt / write_frostt_string."""
    lib = load_library()
    n = C.c_uint64()
    _check(lib.mk_frostt_format(t.mode_count(), t.nnz, _ptr(t.coords), _ptr(t.values),
                                _value_prec(t), threads, None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    _check(lib.mk_frostt_format(t.mode_count(), t.nnz, _ptr(t.coords), _ptr(t.values),
                                _value_prec(t), threads, buf, n.value, C.byref(n)))
    return buf.raw[:n.value].decode()


def write_frostt_file(t: SparseTensorCOO, path, threads: int = 0) -> None:
    """frostt.hpp:201-206 write_frostt_file."""
    _check(load_library().mk_frostt_write_file(os.fsencode(path), t.mode_count(), t.nnz,
                                               _ptr(t.coords), _ptr(t.values), _value_prec(t),
                                               threads))


def save_tensor_cache(t: SparseTensorCOO, path) -> None:
    """Binary tensor cache ("MKBT" v1, checksummed AoS coordinates + values)."""
    d = np.asarray(t.dims, dtype=np.uint32)
    _check(load_library().mk_tensor_cache_write(os.fsencode(path), t.mode_count(), _ptr(d),
                                                t.nnz, _ptr(t.coords), _ptr(t.values),
                                                _value_prec(t)))


def load_tensor_cache(path) -> SparseTensorCOO:
    h = C.c_void_p()
    _check(load_library().mk_tensor_cache_read(os.fsencode(path), C.byref(h)))
    return _take_host_tensor(h)[0]


def load_tensor(path, options: Optional[FrosttOptions] = None, dtype=np.float32,
                cache: bool = True) -> FrosttParseResult:
    """A FROSTT file through the binary cache `<path>.mkbt`: the cache is used when it is
    newer than the text and was written with the same precision (else the text is parsed
    and the cache rewritten).  The cache stores the parse result, so duplicates_merged of a
    cached load is reported as 0."""
    cpath = os.fspath(path) + ".mkbt"
    if cache and options is None and os.path.exists(cpath) and \
            os.path.getmtime(cpath) >= os.path.getmtime(path):
        try:
            t = load_tensor_cache(cpath)
            if t.values.dtype == np.dtype(dtype):
                return FrosttParseResult(t, 0)
        except MttkrpError:
            pass  # stale or corrupt cache: re-parse below
    res = read_frostt_file(path, options, dtype)
    if cache and options is None:
        try:
            save_tensor_cache(res.tensor, cpath)
        except MttkrpError:
            pass  # read-only location: the parse result is still returned
    return res


def shard_split(row_ptr, world: int) -> np.ndarray:
    """mk_shard_split: the element cut points of mk_set_shard (heavy rows split) (host)."""
    lib = load_library()
    rp = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.uint32))
    cuts = np.empty(world + 1, dtype=np.uint64)
    _check(lib.mk_shard_split(_ptr(rp), rp.size - 1, world, _ptr(cuts)))
    return cuts


def shard_cuts(row_ptr, world: int) -> np.ndarray:
    """mk_shard_cuts: copy-row cut points of a CSR row pointer for `world` ranks (host)."""
    lib = load_library()
    rp = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.uint32))
    cuts = np.empty(world + 1, dtype=np.uint64)
    _check(lib.mk_shard_cuts(_ptr(rp), rp.size - 1, world, _ptr(cuts)))
    return cuts


# ----------------------------------------------------------------------------- verify
def verify_against(got, want):
    """verify.hpp:21-39: (max_rel_err, worst_row, worst_col) with |g-w|/max(1,|w|)."""
    g = np.asarray(got.data if isinstance(got, FactorMatrix) else got, dtype=np.float64)
    w = np.asarray(want.data if isinstance(want, FactorMatrix) else want, dtype=np.float64)
    if g.shape != w.shape:
        raise MttkrpError("verify: matrix shapes differ")
    if g.size == 0:
        return 0.0, 0, 0
    err = np.abs(g - w) / np.maximum(1.0, np.abs(w))
    k = int(np.argmax(err))
    return float(err.reshape(-1)[k]), k // g.shape[1], k % g.shape[1]


def verify_tolerance(dtype=np.float32) -> float:
    """verify.hpp:42-45."""
    return 1e-5 if np.dtype(dtype).itemsize == 4 else 1e-12
