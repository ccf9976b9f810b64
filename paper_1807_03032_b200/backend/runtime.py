"""ctypes binding of the C ABI (include/stencil_b200.h).

The shared library is built in-tree (csrc/Makefile -> libstencil_b200.so).
There is no fallback: if the library or a GPU is missing, execution raises
``BackendError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .buffers import BackendError

LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "libstencil_b200.so")

MAX_FIELDS, MAX_DENSE, MAX_SPARSE = 16, 4, 16
MAX_CORNERS, MAX_FACTORS, MAX_TABLES, MAX_STAGES = 8, 8, 16, 24

EXPORTS = ("sc_version", "sc_last_error", "sc_device_count", "sc_set_device",
           "sc_run", "sc_plan_size", "sc_prepare", "sc_launch", "sc_release",
           "sc_step", "sc_step_part", "sc_measure_fp32", "sc_revalidate",
           "sc_upload_shell", "sc_early_download",
           "sc_multi_unique_id", "sc_multi_init", "sc_multi_finalize",
           "sc_multi_run", "sc_multi_exchange")


class ScField(C.Structure):
    _fields_ = [("data", C.c_void_p), ("ext", C.c_int64 * 4),
                ("ndim", C.c_int32), ("nslots", C.c_int32),
                ("has_time", C.c_int32), ("pad", C.c_int32)]


class ScOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("dst", C.c_int32), ("a", C.c_int32),
                ("b", C.c_int32)]


class ScLoad(C.Structure):
    _fields_ = [("field", C.c_int32), ("tshift", C.c_int32),
                ("off", C.c_int32 * 3), ("tdiv", C.c_int32)]


class ScDense(C.Structure):
    _fields_ = [("nops", C.c_int32), ("nloads", C.c_int32),
                ("nconsts", C.c_int32), ("out_reg", C.c_int32),
                ("nregs", C.c_int32),
                ("ops", C.POINTER(ScOp)), ("loads", C.POINTER(ScLoad)),
                ("consts", C.POINTER(C.c_double)),
                ("target", ScLoad), ("fast_kind", C.c_int32),
                ("so", C.c_int32), ("has_damp", C.c_int32),
                ("u_field", C.c_int32), ("m_field", C.c_int32),
                ("damp_field", C.c_int32), ("nfast_consts", C.c_int32),
                ("fast_consts", C.POINTER(C.c_double)),
                ("tti_fields", C.c_int32 * 8), ("exec_kind", C.c_int32),
                ("tguard", C.c_int32), ("xblock", C.c_int32),
                ("scratch", C.c_void_p * 6),
                ("iblock", C.c_int32), ("jblock", C.c_int32)]


class ScSparse(C.Structure):
    _fields_ = [("kind", C.c_int32), ("npoint", C.c_int32),
                ("ncorner", C.c_int32), ("ndim", C.c_int32),
                ("base", C.c_void_p),
                ("delta", (C.c_int32 * 3) * MAX_CORNERS),
                ("nfac", C.c_int32 * MAX_CORNERS),
                ("fac_kind", (C.c_int32 * MAX_FACTORS) * MAX_CORNERS),
                ("fac_arg", (C.c_int32 * MAX_FACTORS) * MAX_CORNERS),
                ("fac_const", (C.c_double * MAX_FACTORS) * MAX_CORNERS),
                ("lead", C.c_double * MAX_CORNERS),
                ("tables", C.c_void_p * MAX_TABLES),
                ("field", C.c_int32), ("field_tshift", C.c_int32),
                ("sparse", C.c_void_p), ("sparse_nt", C.c_int64),
                ("sparse_tshift", C.c_int32), ("serial", C.c_int32)]


class ScPlan(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("ndim", C.c_int32),
                ("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3),
                ("t_m", C.c_int32), ("t_M", C.c_int32),
                ("nfields", C.c_int32), ("fields", ScField * MAX_FIELDS),
                ("ndense", C.c_int32), ("dense", ScDense * MAX_DENSE),
                ("nsparse", C.c_int32), ("sparse", ScSparse * MAX_SPARSE),
                ("nstages", C.c_int32), ("stages", C.c_int32 * MAX_STAGES),
                ("stream", C.c_void_p),
                ("stage_ms", C.c_float * MAX_STAGES),
                ("launches", C.c_int32), ("profile", C.c_int32),
                ("total_ms", C.c_float), ("pad3", C.c_int32)]


class ScExchange(C.Structure):
    """sc_exchange: the ghost-plane exchange of one x-slab rank."""
    _fields_ = [("nfields", C.c_int32), ("field", C.c_int32 * 4),
                ("lo_peer", C.c_int32), ("hi_peer", C.c_int32),
                ("halo", C.c_int32), ("slab", C.c_int32),
                ("overlap", C.c_int32), ("nearly", C.c_int32),
                ("early", (C.c_int32 * 2) * 2), ("interior", C.c_int32 * 2),
                ("n_early_points", C.c_int32), ("pad", C.c_int32)]


_lib = None
_lock = threading.Lock()


def load_library(path: str = None):
    """Load and sanity-check the C ABI (no GPU needed). ``SC_LIB_PATH``
    selects another in-tree build (A/B kernel experiments)."""
    global _lib
    path = path or os.environ.get("SC_LIB_PATH") or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise BackendError("B200 backend library missing: %s (run "
                               "__graft_entry__.build())" % path)
        lib = C.CDLL(path)
        for name in EXPORTS:
            if not hasattr(lib, name):
                raise BackendError("library lacks export %s" % name)
        lib.sc_last_error.restype = C.c_char_p
        lib.sc_plan_size.restype = C.c_int64
        lib.sc_run.argtypes = [C.POINTER(ScPlan)]
        lib.sc_device_count.argtypes = [C.POINTER(C.c_int)]
        lib.sc_prepare.argtypes = [C.POINTER(ScPlan), C.POINTER(C.c_void_p)]
        lib.sc_launch.argtypes = [C.c_void_p, C.POINTER(ScPlan)]
        lib.sc_release.argtypes = [C.c_void_p]
        lib.sc_step.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        lib.sc_revalidate.argtypes = [C.c_void_p, C.c_void_p]
        lib.sc_multi_unique_id.argtypes = [C.c_void_p]
        lib.sc_multi_init.argtypes = [C.c_void_p, C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p)]
        lib.sc_multi_finalize.argtypes = [C.c_void_p]
        lib.sc_multi_run.argtypes = [C.c_void_p, C.c_void_p,
                                     C.POINTER(ScExchange), C.c_void_p]
        lib.sc_multi_exchange.argtypes = [C.c_void_p, C.c_void_p,
                                          C.POINTER(ScExchange), C.c_int,
                                          C.c_void_p]
        lib.sc_measure_fp32.argtypes = [C.POINTER(C.c_double)]
        lib.sc_early_download.argtypes = [C.c_void_p, C.c_int, C.c_void_p,
                                          C.c_void_p, C.c_int64]
        lib.sc_upload_shell.argtypes = [C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.c_int,
                                        C.c_void_p]
        lib.sc_step_part.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                     C.c_int, C.c_int, C.c_int, C.c_int]
        if lib.sc_plan_size() != C.sizeof(ScPlan):
            raise BackendError("sc_plan layout mismatch: C %d vs ctypes %d"
                               % (lib.sc_plan_size(), C.sizeof(ScPlan)))
        _lib = lib
        return lib


def last_error() -> str:
    lib = load_library()
    msg = lib.sc_last_error()
    return msg.decode() if msg else ""


def measure_fp32_tflops() -> float:
    """Dense FP32 TFLOP/s measured on the current device (sc_measure_fp32)."""
    lib = load_library()
    v = C.c_double(0.0)
    if lib.sc_measure_fp32(C.byref(v)) != 0:
        raise BackendError("B200 kernel failure: %s" % last_error())
    return float(v.value)


def run_plan(plan: ScPlan) -> None:
    lib = load_library()
    if lib.sc_run(C.byref(plan)) != 0:
        raise BackendError("B200 kernel failure: %s" % last_error())


class PreparedRun:
    """A prepared C-side run (sc_prepare): launched any number of times."""

    def __init__(self, plan: ScPlan):
        lib = load_library()
        self._lib = lib
        self.handle = C.c_void_p()
        if lib.sc_prepare(C.byref(plan), C.byref(self.handle)) != 0:
            raise BackendError("B200 prepare failed: %s" % last_error())

    def launch(self, plan: ScPlan) -> None:
        if self._lib.sc_launch(self.handle, C.byref(plan)) != 0:
            raise BackendError("B200 kernel failure: %s" % last_error())

    def early_download(self, t_split: int, dev: int, host: int,
                       nbytes: int) -> bool:
        """sc_early_download: arm (or, nbytes = 0, disarm) the copy that
        starts once the steps before t_split are done."""
        rc = self._lib.sc_early_download(self.handle, int(t_split),
                                         C.c_void_p(dev), C.c_void_p(host),
                                         int(nbytes))
        if rc < 0:
            raise BackendError("B200 early download failed: %s" % last_error())
        return rc == 0

    def revalidate(self, stream: int) -> bool:
        """sc_revalidate: the fused kernels' data-dependent preconditions
        still hold on the current device buffers."""
        rc = self._lib.sc_revalidate(self.handle, C.c_void_p(stream))
        if rc < 0:
            raise BackendError("B200 revalidate failed: %s" % last_error())
        return rc == 0

    def step(self, t: int, stream: int) -> None:
        if self._lib.sc_step(self.handle, int(t), C.c_void_p(stream)) != 0:
            raise BackendError("B200 kernel failure: %s" % last_error())

    def step_part(self, t: int, stream: int, x_lo: int, x_hi: int,
                  p_lo: int, p_hi: int, what: int) -> None:
        if self._lib.sc_step_part(self.handle, int(t), C.c_void_p(stream),
                                  int(x_lo), int(x_hi), int(p_lo), int(p_hi),
                                  int(what)) != 0:
            raise BackendError("B200 kernel failure: %s" % last_error())

    def multi_run(self, comm: "MultiComm", x: ScExchange, stream: int) -> None:
        """sc_multi_run: the whole slab t loop with the ghost exchange."""
        h = comm.handle if comm is not None else None
        if self._lib.sc_multi_run(self.handle, h, C.byref(x),
                                  C.c_void_p(stream)) != 0:
            raise BackendError("B200 multi-GPU run failed: %s" % last_error())

    def multi_exchange(self, comm: "MultiComm", x: ScExchange, t: int,
                       stream: int) -> None:
        h = comm.handle if comm is not None else None
        if self._lib.sc_multi_exchange(self.handle, h, C.byref(x), int(t),
                                       C.c_void_p(stream)) != 0:
            raise BackendError("B200 ghost exchange failed: %s" % last_error())

    def close(self) -> None:
        if self.handle:
            self._lib.sc_release(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def multi_unique_id() -> bytes:
    """sc_multi_unique_id: a fresh NCCL unique id (128 bytes, rank 0)."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    if lib.sc_multi_unique_id(buf) != 0:
        raise BackendError("NCCL unique id failed: %s" % last_error())
    return buf.raw


class MultiComm:
    """An NCCL communicator of the library's multi-GPU data plane
    (sc_multi_init / sc_multi_finalize)."""

    def __init__(self, uid: bytes, rank: int, world: int):
        lib = load_library()
        self._lib = lib
        self.handle = C.c_void_p()
        self.rank, self.world = rank, world
        if lib.sc_multi_init(C.create_string_buffer(uid, 128), int(rank),
                             int(world), C.byref(self.handle)) != 0:
            raise BackendError("sc_multi_init failed: %s" % last_error())

    def close(self) -> None:
        if self.handle:
            self._lib.sc_multi_finalize(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
