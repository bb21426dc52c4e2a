"""ctypes binding of libvqc.so (include/vqc.h) — the only compute path.

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, the first call raises. Device buffers are torch CUDA tensors
(torch supplies memory, streams and the caching allocator); only raw pointers
and sizes cross the C ABI.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libvqc.so")

_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p

VQC_MODE_FORWARD, VQC_MODE_VJP, VQC_MODE_JACOBIAN = 0, 1, 2
# state precision of a plan (vqc_plan_create's precision argument)
PRECISIONS = {"complex128": 0, "complex64": 1}
_ERRORS = {-1: ValueError, -2: NotImplementedError, -3: RuntimeError, -4: RuntimeError,
           -5: MemoryError}

EXPORTED_SYMBOLS = (
    "vqc_plan_create", "vqc_plan_destroy", "vqc_plan_num_cols", "vqc_plan_num_obs",
    "vqc_plan_mode", "vqc_plan_describe", "vqc_workspace_bytes", "vqc_forward", "vqc_adjoint",
    "vqc_run_batch_host", "vqc_last_launch_count", "vqc_profile_enable", "vqc_profile_report",
    "vqc_last_error", "vqc_abi_version", "vqc_jit_source", "vqc_spsa_signs",
)


class VqcCircuit(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("n_gates", ctypes.c_int64),
                ("kinds", _I64P), ("q0", _I64P), ("q1", _I64P), ("coeff", _F64P),
                ("f_offs", _I64P), ("f_idx", _I64P), ("total_params", ctypes.c_int64),
                ("enc_offset", ctypes.c_int64), ("enc_size", ctypes.c_int64)]


class VqcObservables(ctypes.Structure):
    _fields_ = [("n_obs", ctypes.c_int64), ("term_offs", _I64P), ("coeffs", _F64P),
                ("x_masks", _I64P), ("sign_masks", _I64P), ("phases", _F64P)]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | None = None):
    """Load libvqc.so once; raises if it has not been built."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = path or LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(f"libvqc.so not found at {path}; run __graft_entry__.build() "
                               "(the GPU path has no CPU fallback)")
        lib = ctypes.CDLL(path)
        lib.vqc_plan_create.restype = ctypes.c_int
        lib.vqc_plan_create.argtypes = [ctypes.POINTER(VqcCircuit), ctypes.POINTER(VqcObservables),
                                        _I64P, ctypes.c_int, ctypes.POINTER(_VP)]
        lib.vqc_plan_destroy.restype = None
        lib.vqc_plan_destroy.argtypes = [_VP]
        for name in ("vqc_plan_num_cols", "vqc_plan_num_obs"):
            getattr(lib, name).restype = ctypes.c_int64
            getattr(lib, name).argtypes = [_VP]
        lib.vqc_plan_mode.restype = ctypes.c_int
        lib.vqc_plan_mode.argtypes = [_VP]
        lib.vqc_plan_describe.restype = ctypes.c_int64
        lib.vqc_plan_describe.argtypes = [_VP, ctypes.c_char_p, ctypes.c_int64]
        lib.vqc_workspace_bytes.restype = ctypes.c_size_t
        lib.vqc_workspace_bytes.argtypes = [_VP, ctypes.c_int64, ctypes.c_int]
        lib.vqc_forward.restype = ctypes.c_int
        lib.vqc_forward.argtypes = [_VP, _VP, _VP, ctypes.c_int64, _VP, _VP, ctypes.c_size_t, _VP]
        lib.vqc_adjoint.restype = ctypes.c_int
        lib.vqc_adjoint.argtypes = [_VP, _VP, _VP, ctypes.c_int64, _VP, _VP, _VP, _VP, _VP, _VP,
                                    ctypes.c_size_t, _VP]
        lib.vqc_run_batch_host.restype = ctypes.c_int
        lib.vqc_run_batch_host.argtypes = [_VP, _F64P, _F64P, ctypes.c_int64, _F64P, _F64P, _F64P,
                                           _F64P, _F64P]
        lib.vqc_jit_source.restype = ctypes.c_int64
        lib.vqc_jit_source.argtypes = [ctypes.POINTER(VqcCircuit), _I64P, ctypes.c_int, ctypes.c_char_p,
                                       ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]
        lib.vqc_spsa_signs.restype = ctypes.c_int
        lib.vqc_spsa_signs.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int, _VP]
        lib.vqc_last_launch_count.restype = ctypes.c_int64
        lib.vqc_last_launch_count.argtypes = []
        lib.vqc_profile_enable.restype = None
        lib.vqc_profile_enable.argtypes = [ctypes.c_int]
        lib.vqc_profile_report.restype = ctypes.c_int64
        lib.vqc_profile_report.argtypes = [ctypes.c_char_p, ctypes.c_int64]
        lib.vqc_last_error.restype = ctypes.c_char_p
        lib.vqc_last_error.argtypes = []
        lib.vqc_abi_version.restype = ctypes.c_int
        lib.vqc_abi_version.argtypes = []
        _lib = lib
        return lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().vqc_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(f"{what}: {msg}")


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Plan:
    """Owns one VqcPlan* (device tables for one circuit/observables/wrt)."""

    def __init__(self, compiled, pack, wrt_col, enc_offset: int, enc_size: int, device=None,
                 precision: str = "complex128"):
        import torch  # noqa: F401  (CUDA context on the right device)

        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(PRECISIONS)}, got {precision!r}")
        self.precision = precision

        lib = load_library()
        self._keep = [_i64(compiled.kinds), _i64(compiled.q0), _i64(compiled.q1),
                      _f64(compiled.coeff), _i64(compiled.f_offs),
                      _i64(compiled.f_idx if len(compiled.f_idx) else np.zeros(1, np.int64)),
                      _i64(pack.term_offs),
                      _f64(pack.coeffs if len(pack.coeffs) else np.zeros(1)),
                      _i64(pack.x_masks if len(pack.x_masks) else np.zeros(1, np.int64)),
                      _i64(pack.sign_masks if len(pack.sign_masks) else np.zeros(1, np.int64)),
                      _f64(pack.phases.reshape(-1) if pack.phases.size else np.zeros(2)),
                      _i64(wrt_col if len(wrt_col) else np.zeros(1, np.int64))]
        k = self._keep
        circ = VqcCircuit(compiled.num_qubits, len(compiled.kinds),
                          k[0].ctypes.data_as(_I64P), k[1].ctypes.data_as(_I64P),
                          k[2].ctypes.data_as(_I64P), k[3].ctypes.data_as(_F64P),
                          k[4].ctypes.data_as(_I64P), k[5].ctypes.data_as(_I64P),
                          compiled.total_params, enc_offset, enc_size)
        obs = VqcObservables(pack.num_obs, k[6].ctypes.data_as(_I64P), k[7].ctypes.data_as(_F64P),
                             k[8].ctypes.data_as(_I64P), k[9].ctypes.data_as(_I64P),
                             k[10].ctypes.data_as(_F64P))
        self.device = device
        handle = _VP()
        if device is not None:
            import torch
            with torch.cuda.device(device):
                rc = lib.vqc_plan_create(ctypes.byref(circ), ctypes.byref(obs),
                                         k[11].ctypes.data_as(_I64P), PRECISIONS[precision],
                                         ctypes.byref(handle))
        else:
            rc = lib.vqc_plan_create(ctypes.byref(circ), ctypes.byref(obs),
                                     k[11].ctypes.data_as(_I64P), PRECISIONS[precision],
                                     ctypes.byref(handle))
        _check(rc, "vqc_plan_create")
        self._h = handle
        self._lib = lib
        self.num_cols = int(lib.vqc_plan_num_cols(handle))
        self.num_obs = int(lib.vqc_plan_num_obs(handle))
        self.mode = int(lib.vqc_plan_mode(handle))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.vqc_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(1024)
        self._lib.vqc_plan_describe(self._h, buf, 1024)
        return buf.value.decode()

    def workspace_bytes(self, B: int, mode: int) -> int:
        return int(self._lib.vqc_workspace_bytes(self._h, B, mode))

    def forward(self, inputs, weights, expect, workspace, stream) -> None:
        ws_bytes = workspace.numel() if workspace is not None else 0
        _check(self._lib.vqc_forward(self._h, _ptr(inputs), _ptr(weights), inputs.shape[0],
                                     _ptr(expect), _ptr(workspace), ws_bytes, stream),
               "vqc_forward")

    def adjoint(self, inputs, weights, upstream, expect, jac, vjp_rows, vjp_sum, workspace,
                stream) -> None:
        ws_bytes = workspace.numel() if workspace is not None else 0
        _check(self._lib.vqc_adjoint(self._h, _ptr(inputs), _ptr(weights), inputs.shape[0],
                                     _ptr(upstream), _ptr(expect), _ptr(jac), _ptr(vjp_rows),
                                     _ptr(vjp_sum), _ptr(workspace), ws_bytes, stream),
               "vqc_adjoint")

    def run_batch_host(self, inputs: np.ndarray, weights: np.ndarray, upstream=None,
                       jacobian: bool = False, out=None):
        """numpy in / numpy out through vqc_run_batch_host (H2D + run + D2H).
        ``out``: optional preallocated (expect, rows, vsum) arrays (e.g. views of
        pinned host memory)."""
        inputs = _f64(inputs)
        weights = _f64(weights)
        B = inputs.shape[0]
        M, C = self.num_obs, self.num_cols
        if out is not None:
            expect, rows, vsum = out
            jac = None
        else:
            expect = np.empty((B, M))
            jac = np.empty((B, M, C)) if jacobian else None
            rows = np.empty((B, C)) if upstream is not None else None
            vsum = np.empty(C) if upstream is not None else None
        up = _f64(upstream) if upstream is not None else None

        def p(a):
            return None if a is None else a.ctypes.data_as(_F64P)

        _check(self._lib.vqc_run_batch_host(self._h, p(inputs), p(weights), B, p(up), p(expect),
                                            p(jac), p(rows), p(vsum)), "vqc_run_batch_host")
        return expect, jac, rows, vsum


def jit_source(compiled, wrt_col, enc_offset: int, enc_size: int, compile: bool = False):
    """(CUDA source, NVRTC compile seconds or None) of the kernels a plan for
    this circuit would JIT-compile; runs on the CPU (no device needed)."""
    lib = load_library()
    keep = [_i64(compiled.kinds), _i64(compiled.q0), _i64(compiled.q1), _f64(compiled.coeff),
            _i64(compiled.f_offs), _i64(compiled.f_idx if len(compiled.f_idx) else np.zeros(1, np.int64)),
            _i64(wrt_col if len(wrt_col) else np.zeros(1, np.int64))]
    circ = VqcCircuit(compiled.num_qubits, len(compiled.kinds), keep[0].ctypes.data_as(_I64P),
                      keep[1].ctypes.data_as(_I64P), keep[2].ctypes.data_as(_I64P),
                      keep[3].ctypes.data_as(_F64P), keep[4].ctypes.data_as(_I64P),
                      keep[5].ctypes.data_as(_I64P), compiled.total_params, enc_offset, enc_size)
    secs = ctypes.c_double(0.0)
    n = lib.vqc_jit_source(ctypes.byref(circ), keep[6].ctypes.data_as(_I64P), 1 if compile else 0, None, 0,
                           ctypes.byref(secs))
    _check(int(n) if n < 0 else 0, "vqc_jit_source")
    buf = ctypes.create_string_buffer(int(n) + 1)
    lib.vqc_jit_source(ctypes.byref(circ), keep[6].ctypes.data_as(_I64P), 0, buf, int(n) + 1, None)
    return buf.value.decode(), (secs.value if compile else None)


def spsa_signs(seed: int, row0: int, rows: int, samples: int, cols: int,
               per_row_seed: bool = True) -> np.ndarray:
    """(rows, samples, cols) int8 of +-1: the reference's per-row SPSA draws
    (numpy default_rng(mix_seed(seed, row)).integers(0, 2, size=cols) per
    sample), generated natively on the host."""
    out = np.empty((rows, samples, cols), np.int8)
    _check(load_library().vqc_spsa_signs(int(seed) & 0xFFFFFFFFFFFFFFFF, int(row0), int(rows), int(samples),
                                         int(cols), 1 if per_row_seed else 0, out.ctypes.data),
           "vqc_spsa_signs")
    return out


def last_launch_count() -> int:
    return int(load_library().vqc_last_launch_count())


def profile_enable(on: bool = True) -> None:
    """Per-kernel CUDA-event timing of this thread's launches (resets totals)."""
    load_library().vqc_profile_enable(1 if on else 0)


def profile_report() -> dict:
    """{kernel: (total_ms, launches)} for launches since profile_enable."""
    import json
    lib = load_library()
    n = int(lib.vqc_profile_report(None, 0))
    buf = ctypes.create_string_buffer(n + 1)
    lib.vqc_profile_report(buf, n + 1)
    return {k: (float(v[0]), int(v[1])) for k, v in json.loads(buf.value.decode()).items()}
