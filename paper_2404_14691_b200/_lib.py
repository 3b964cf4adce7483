"""ctypes binding of libsagedp.so (include/sage_dp.h).

This is the product path: there is no fallback.  If the shared library is
missing the import of `lib()` raises, and every data-plane call fails loudly.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libsagedp.so"

SAGE_OK = 0
SAGE_EINVAL = -1
SAGE_ENOMEM = -2
SAGE_ECUDA = -3
SAGE_ENOTREADY = -4
SAGE_ESTATE = -5
SAGE_ECHECKSUM = -6
SAGE_ENODEV = -7

SAGE_INIT_PEER_ACCESS = 0x1
SAGE_INIT_SHARE_DEVICE = 0x2
CLASS_CONTEXT, CLASS_READ_ONLY, CLASS_WRITABLE, CLASS_INSTANCE_FIXED = 0, 1, 2, 3
ALLOC_ACCOUNT_ONLY = 0x100
LOAD_SRC_PINNED, LOAD_SRC_DEVICE, LOAD_SRC_PEER, LOAD_NO_VERIFY = 0x1, 0x2, 0x4, 0x8
BODY_TOUCH, BODY_SGEMM, BODY_STENCIL, BODY_SPMV, BODY_SPIN, BODY_SGEMM_F32, BODY_GATHER = 0, 1, 2, 3, 4, 5, 6
BODY_SPMV_CSB = 7

u64 = C.c_uint64
i64 = C.c_int64
H = C.c_uint64  # sage_handle


class SageError(RuntimeError):
    def __init__(self, code: int, what: str, msg: str):
        super().__init__(f"{what} failed ({code}): {msg}")
        self.code = code


class LoadDesc(C.Structure):
    _fields_ = [("gpu", C.c_int32), ("flags", C.c_uint32), ("dst", u64), ("layout", H),
                ("src", C.c_void_p), ("src_bytes", u64), ("wait", C.POINTER(H)), ("n_wait", C.c_int32),
                ("src_gpu", C.c_int32)]


class LoadInfo(C.Structure):
    _fields_ = [("cpu_begin_us", i64), ("cpu_end_us", i64), ("gpu_begin_us", i64), ("gpu_end_us", i64),
                ("host_bytes", u64), ("link_bytes", u64), ("landed_bytes", u64), ("checksum", u64),
                ("chunks", C.c_uint32), ("status", C.c_int32)]


class BodyDesc(C.Structure):
    _fields_ = [("body", C.c_int32), ("pad_", C.c_int32), ("ro", u64), ("input", u64), ("out", u64),
                ("ro_bytes", u64), ("input_bytes", u64), ("out_bytes", u64), ("args", i64 * 8)]


INSTANCE_THREAD, INSTANCE_PROCESS, INSTANCE_POOLED = 0, 1, 2


class FixedGSLDesc(C.Structure):
    _fields_ = [("gpu", C.c_int32), ("mode", C.c_int32), ("layout", H), ("ro_src", C.c_void_p),
                ("ro_src_bytes", u64), ("input", C.c_void_p), ("input_bytes", u64), ("alloc_bytes", u64),
                ("body", BodyDesc), ("result", C.c_void_p), ("result_bytes", u64), ("ctx", H)]


INV_CTX, INV_RO, INV_INPUT, INV_SYNC, INV_RET_HOST, INV_VERIFY_INPUT = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
SRC_HOST, SRC_PINNED, SRC_HBM, SRC_PEER = 0, 1, 2, 3


class InvokeDesc(C.Structure):
    _fields_ = [("gpu", C.c_int32), ("flags", C.c_uint32), ("ctx_dptr", u64), ("ctx_bytes", u64),
                ("ro_kind", C.c_int32), ("ro_src_gpu", C.c_int32), ("ro_layout", H), ("ro_src", C.c_void_p),
                ("ro_src_bytes", u64), ("ro_dst", u64), ("ro_wait", H * 2), ("n_ro_wait", C.c_int32),
                ("in_kind", C.c_int32), ("in_src", C.c_void_p), ("in_bytes", u64), ("in_dst", u64),
                ("wait", H * 4), ("n_wait", C.c_int32), ("pad_", C.c_int32), ("body", BodyDesc),
                ("ret_src", u64), ("ret_dst", C.c_void_p), ("ret_bytes", u64)]


class InvokeInfo(C.Structure):
    _fields_ = [("t", i64 * 16), ("host_bytes", u64), ("link_bytes", u64), ("ro_checksum", u64),
                ("in_checksum", u64), ("ro_landed_us", i64), ("status", C.c_int32), ("pad_", C.c_int32)]


class FixedGSLInfo(C.Structure):
    _fields_ = [("t", i64 * 16), ("checksum", u64), ("teardown_us", i64), ("status", C.c_int32),
                ("pad_", C.c_int32)]


SHARE_RO, SHARE_CTX, SHARE_MULTI_STAGE = 0x1, 0x2, 0x4
FN_HAS_RO = 0x1
ADMIT_DEFER_RO_LEADER, ADMIT_DEFERRED = 0x1, 1
TOKEN_RO, TOKEN_CTX = 0, 1
STEP_CACHE_RO, STEP_FREE_RO, STEP_FREE_CTX, STEP_DROP_CACHE = 0x01, 0x02, 0x04, 0x08
STEP_EVICT, STEP_GPU_FREED, STEP_ARM = 0x10, 0x20, 0x40
HOLD_RO, HOLD_CTX, HOLD_CACHE, HOLD_CPU_CTX, HOLD_CONTAINER = 0x1, 0x2, 0x4, 0x8, 0x10


class ShareGrant(C.Structure):
    _fields_ = [("warmth", C.c_int32), ("shared_ro", C.c_uint8), ("shared_ctx", C.c_uint8),
                ("wait_ro", C.c_uint8), ("wait_ctx", C.c_uint8), ("leader_ro", C.c_uint8),
                ("leader_ctx", C.c_uint8), ("timer_cancelled", C.c_uint8), ("new_resident", C.c_uint8),
                ("alloc_ro", u64), ("alloc_ctx", u64), ("resident", u64)]


class ShareStep(C.Structure):
    _fields_ = [("actions", C.c_uint32), ("state_before", C.c_int32), ("state_after", C.c_int32),
                ("timer_gen", C.c_uint32), ("timer_cancelled", C.c_uint8), ("pad_", C.c_uint8 * 7),
                ("deadline_us", i64), ("resident", u64)]


class ResidentInfo(C.Structure):
    _fields_ = [("resident", u64), ("fn", C.c_int32), ("gpu", C.c_int32), ("state", C.c_int32),
                ("active", C.c_uint32), ("holds", C.c_uint32), ("timer_gen", C.c_uint32),
                ("ro_bytes", u64), ("ctx_bytes", u64), ("last_activity_us", i64), ("deadline_us", i64),
                ("has_checksum", C.c_uint32), ("pad_", C.c_uint32), ("checksum", u64)]


CONV_NHWC, CONV_C4, CONV_S2D = 0, 1, 2
BODY_RESNET50 = 8
NET_PAD_INPUT, NET_CONV, NET_MAXPOOL, NET_POOL_FC, NET_S2D_INPUT = 1, 2, 3, 4, 5
NET_BUF_INPUT, NET_BUF_OUT, NET_BUF_WS0 = 0, 1, 2


class NetOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("src", C.c_int32), ("dst", C.c_int32), ("res", C.c_int32),
                ("w_off", u64), ("g_off", u64), ("b_off", u64), ("m_off", u64), ("v_off", u64),
                ("eps", C.c_float), ("n", C.c_int32), ("h", C.c_int32), ("w", C.c_int32), ("cin", C.c_int32),
                ("cout", C.c_int32), ("r", C.c_int32), ("s", C.c_int32), ("stride", C.c_int32),
                ("pad", C.c_int32), ("relu", C.c_int32), ("mode", C.c_int32)]


class ConvDesc(C.Structure):
    _fields_ = [("x", u64), ("w", u64), ("out", u64), ("residual", u64), ("bn_gamma", u64), ("bn_beta", u64),
                ("bn_mean", u64), ("bn_var", u64), ("bn_eps", C.c_float), ("n", C.c_int32), ("h", C.c_int32),
                ("w_", C.c_int32), ("cin", C.c_int32), ("cout", C.c_int32), ("r", C.c_int32), ("s", C.c_int32),
                ("stride", C.c_int32), ("pad", C.c_int32), ("relu", C.c_int32), ("mode", C.c_int32),
                ("pad_", C.c_int32)]


BCAST_P2P_ONLY, BCAST_PATH_P2P, BCAST_PATH_MULTICAST = 0x1, 0, 1


class FanoutCaps(C.Structure):
    _fields_ = [("n_gpus", C.c_int32), ("n_devices", C.c_int32), ("peer_mask", C.c_uint32 * 32),
                ("multicast_attr", C.c_int32), ("multicast", C.c_int32), ("multicast_granularity", u64),
                ("why", C.c_char * 160)]


class BcastDesc(C.Structure):
    _fields_ = [("src_gpu", C.c_int32), ("n_dst", C.c_int32), ("src_dptr", u64), ("bytes", u64),
                ("dst_gpu", C.c_int32 * 32), ("dst_alloc", H * 32), ("flags", C.c_uint32), ("path", C.c_int32)]


_SIGS = {
    "sage_init": (C.c_int, [C.c_int, u64, u64, u64, C.c_uint32]),
    "sage_shutdown": (C.c_int, []),
    "sage_last_error": (C.c_char_p, []),
    "sage_abi_version": (C.c_int, []),
    "sage_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "sage_gpu_device": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "sage_now_us": (i64, []),
    "sage_clock_epoch_ns": (i64, []),
    "sage_set_host_threads": (C.c_int, [C.c_int]),
    "sage_pool_configure": (C.c_int, [C.c_int, u64, u64]),
    "sage_pool_alloc": (C.c_int, [C.c_int, u64, C.c_int, C.POINTER(H), C.POINTER(u64), C.POINTER(u64)]),
    "sage_pool_free": (C.c_int, [H]),
    "sage_pool_free_after": (C.c_int, [H, H]),
    "sage_pool_free_after_n": (C.c_int, [H, C.POINTER(H), C.c_int]),
    "sage_pool_effective": (C.c_int, [C.c_int, u64, C.POINTER(u64)]),
    "sage_pool_usage": (C.c_int, [C.c_int, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    "sage_pool_trim": (C.c_int, [C.c_int, C.POINTER(u64)]),
    "sage_pool_dptr": (C.c_int, [H, C.POINTER(u64), C.POINTER(u64)]),
    "sage_host_alloc": (C.c_int, [u64, C.POINTER(H), C.POINTER(C.c_void_p)]),
    "sage_host_free": (C.c_int, [H]),
    "sage_host_register": (C.c_int, [C.c_void_p, u64]),
    "sage_host_unregister": (C.c_int, [C.c_void_p]),
    "sage_layout_create": (C.c_int, [C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.c_uint32, u64, u64,
                                     C.POINTER(H)]),
    "sage_layout_destroy": (C.c_int, [H]),
    "sage_layout_chunks": (C.c_int, [H, C.POINTER(C.c_uint32)]),
    "sage_layout_checksum": (C.c_int, [H, C.c_void_p, u64, C.POINTER(u64)]),
    "sage_event_query": (C.c_int, [H]),
    "sage_event_sync": (C.c_int, [H]),
    "sage_event_time": (C.c_int, [H, C.POINTER(i64)]),
    "sage_event_release": (C.c_int, [H]),
    "sage_event_alias": (C.c_int, [H, C.POINTER(H)]),
    "sage_event_poll": (C.c_int, [C.POINTER(H), C.c_int, C.POINTER(C.c_uint8), i64]),
    "sage_ctx_acquire": (C.c_int, [C.c_int, C.POINTER(H)]),
    "sage_ctx_release": (C.c_int, [H]),
    "sage_ctx_bind": (C.c_int, [H, u64, u64, C.POINTER(H), C.c_int, C.POINTER(H), C.POINTER(H)]),
    "sage_stream_wait": (C.c_int, [H, C.POINTER(H), C.c_int]),
    "sage_slot_record": (C.c_int, [H, C.POINTER(H)]),
    "sage_slot_stream": (C.c_int, [H, C.POINTER(u64)]),
    "sage_segment_load": (C.c_int, [C.POINTER(LoadDesc), C.POINTER(H), C.POINTER(H)]),
    "sage_load_info_get": (C.c_int, [H, C.POINTER(LoadInfo)]),
    "sage_load_release": (C.c_int, [H]),
    "sage_host_load": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, u64, C.POINTER(H), C.c_int, C.POINTER(H),
                                 C.POINTER(H)]),
    "sage_segment_checksum": (C.c_int, [C.c_int, u64, u64, C.POINTER(u64)]),
    "sage_d2h_cache": (C.c_int, [C.c_int, u64, C.c_void_p, u64, C.POINTER(H), C.c_int, C.POINTER(H)]),
    "sage_fanout": (C.c_int, [C.c_int, u64, C.c_int, u64, u64, C.POINTER(H), C.c_int, C.POINTER(H)]),
    "sage_pool_export": (C.c_int, [H, C.POINTER(C.c_int), C.POINTER(u64)]),
    "sage_segment_import": (C.c_int, [C.c_int, C.c_int, u64, C.POINTER(H), C.POINTER(u64)]),
    "sage_segment_unimport": (C.c_int, [H]),
    "sage_ipc_event_export": (C.c_int, [H, C.POINTER(H), C.c_void_p]),
    "sage_ipc_event_open": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(H)]),
    "sage_launch": (C.c_int, [H, C.POINTER(BodyDesc), C.POINTER(H), C.POINTER(H)]),
    "sage_launch_after": (C.c_int, [H, C.POINTER(H), C.c_int, C.POINTER(BodyDesc), C.POINTER(H), C.POINTER(H)]),
    "sage_return_after": (C.c_int, [H, C.POINTER(H), C.c_int, u64, C.c_void_p, u64, C.POINTER(H), C.POINTER(H)]),
    "sage_sync_wait": (C.c_int, [H, C.POINTER(H), C.c_int, C.POINTER(H), C.POINTER(H)]),
    "sage_return": (C.c_int, [H, u64, C.c_void_p, u64, C.POINTER(H), C.POINTER(H)]),
    "sage_invoke": (C.c_int, [C.POINTER(InvokeDesc), C.POINTER(H), C.POINTER(H), C.POINTER(H), C.POINTER(H)]),
    "sage_invoke_collect": (C.c_int, [H, C.POINTER(InvokeInfo)]),
    "sage_invoke_release": (C.c_int, [H]),
    "sage_invoke_ready": (C.c_int, [C.POINTER(H), C.c_int, i64]),
    "sage_fixedgsl_submit": (C.c_int, [C.POINTER(FixedGSLDesc), C.POINTER(H), C.POINTER(H)]),
    "sage_fixedgsl_info_get": (C.c_int, [H, C.POINTER(FixedGSLInfo)]),
    "sage_fixedgsl_release": (C.c_int, [H]),
    "sage_instance_ctx_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(H)]),
    "sage_instance_ctx_destroy": (C.c_int, [H]),
    "sage_instance_child": (C.c_int, [C.c_int]),
    "sage_stats_enable": (C.c_int, [C.c_int]),
    "sage_stats_reset": (C.c_int, []),
    "sage_stats_get": (C.c_int, [C.c_int, C.c_int, C.POINTER(u64), C.POINTER(C.c_double), C.POINTER(u64)]),
    "sage_device_sync": (C.c_int, [C.c_int]),
    "sage_mark": (C.c_int, [C.c_int, C.POINTER(H)]),
    "sage_event_elapsed": (C.c_int, [H, H, C.POINTER(C.c_double)]),
    "sage_conv": (C.c_int, [H, C.POINTER(ConvDesc)]),
    "sage_fanout_caps": (C.c_int, [C.POINTER(FanoutCaps)]),
    "sage_fanout_broadcast": (C.c_int, [C.POINTER(BcastDesc), C.POINTER(H), C.c_int, C.POINTER(H)]),
    "sage_net_create": (C.c_int, [C.POINTER(NetOp), C.c_int, C.POINTER(u64), C.c_int, C.POINTER(H), C.POINTER(u64)]),
    "sage_net_destroy": (C.c_int, [H]),
    "sage_share_create": (C.c_int, [C.c_int, C.c_uint32, i64, C.POINTER(i64), C.POINTER(H)]),
    "sage_share_destroy": (C.c_int, [H]),
    "sage_share_preview": (C.c_int, [H, C.c_int32, C.c_int, u64, u64, C.c_uint32, C.POINTER(ShareGrant)]),
    "sage_share_admit": (C.c_int, [H, C.c_int32, C.c_int, u64, u64, C.c_uint32, i64, C.POINTER(ShareGrant)]),
    "sage_share_admit_within": (C.c_int, [H, C.c_int32, C.c_int, u64, u64, C.c_uint32, i64, i64, u64, u64,
                                          C.c_uint32, C.POINTER(ShareGrant)]),
    "sage_share_token": (C.c_int, [H, u64, C.c_int, H]),
    "sage_share_token_ready": (C.c_int, [H, u64, C.c_int, C.POINTER(C.c_int)]),
    "sage_share_release": (C.c_int, [H, C.c_int32, C.c_int, i64, C.POINTER(ShareStep)]),
    "sage_share_expire": (C.c_int, [H, u64, C.c_uint32, i64, C.POINTER(ShareStep)]),
    "sage_share_victim": (C.c_int, [H, C.c_int, C.c_int32, C.POINTER(u64)]),
    "sage_share_demote": (C.c_int, [H, u64, i64, C.POINTER(ShareStep)]),
    "sage_share_evict": (C.c_int, [H, u64, C.POINTER(ShareStep)]),
    "sage_share_info": (C.c_int, [H, u64, C.POINTER(ResidentInfo)]),
    "sage_share_lookup": (C.c_int, [H, C.c_int32, C.c_int, C.POINTER(u64)]),
    "sage_share_list": (C.c_int, [H, C.POINTER(u64), C.c_int, C.POINTER(C.c_int)]),
    "sage_share_ro_loads": (C.c_int, [H, C.c_int32, C.c_int, C.POINTER(C.c_uint32)]),
    "sage_share_set_checksum": (C.c_int, [H, u64, u64]),
    "sage_share_find_content": (C.c_int, [H, C.c_int, u64, C.c_int32, C.POINTER(u64)]),
    "sage_share_check": (C.c_int, [H]),
    "sage_debug_emulate_land": (C.c_int, [H, C.c_void_p, u64, C.c_void_p, u64, C.POINTER(u64)]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libsagedp.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.sage_abi_version() != 1:
            raise RuntimeError("libsagedp ABI mismatch")
        _lib = L
        return L


_generation = 0


def generation() -> int:
    """Bumped by every sage_init: native handles from older generations are dead."""
    return _generation


def init(n_gpus: int = 1, pool_bytes: int = 0, staging_bytes: int = 0, chunk_bytes: int = 0,
         flags: int = 0, host_threads: int | None = None) -> None:
    global _generation
    L = lib()
    check(L.sage_set_host_threads(host_threads or host_threads_default()), "sage_set_host_threads")
    check(L.sage_init(n_gpus, pool_bytes, staging_bytes, chunk_bytes, flags), "sage_init")
    _generation += 1
    global _up, _exit_hook
    _up = True
    if not _exit_hook:
        atexit.register(_shutdown_at_exit)
        _exit_hook = True


_up = False
_exit_hook = False


def _shutdown_at_exit() -> None:
    """A process that exits with the plane up (no Simulation.close) drains
    the device and stops the native threads while the CUDA runtime is still
    alive; Python's atexit runs before the C runtime's exit handlers."""
    if _up:
        try:
            shutdown()
        except Exception:   # noqa: BLE001 - best effort on the way out
            pass


def is_up() -> bool:
    return _up


def gpu_device(gpu: int) -> int:
    """Physical CUDA device of logical GPU `gpu` (the library's own mapping)."""
    d = C.c_int(0)
    check(lib().sage_gpu_device(gpu, C.byref(d)), "sage_gpu_device")
    return d.value


def device_count() -> int:
    n = C.c_int(0)
    lib().sage_device_count(C.byref(n))
    return n.value


def shutdown() -> None:
    global _generation
    check(lib().sage_shutdown(), "sage_shutdown")
    _generation += 1
    global _up
    _up = False


def exported_symbols() -> list[str]:
    return list(_SIGS)


def last_error() -> str:
    return (lib().sage_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str) -> int:
    if rc < 0 and rc != SAGE_ENOTREADY:
        raise SageError(rc, what, last_error())
    return rc


def handles(seq) -> tuple:
    """(array pointer, count) for a sequence of handles (None-safe)."""
    seq = [h for h in (seq or ()) if h]
    if not seq:
        return None, 0
    arr = (H * len(seq))(*seq)
    return arr, len(seq)


def host_threads_default() -> int:
    """CPU_LOAD memcpy fan-out: one host thread moves ~3-5 GB/s, PCIe Gen5
    takes ~55 GB/s, so use most cores (leave a few for the control loop)."""
    n = os.cpu_count() or 4
    return max(2, min(16, n - 4))
