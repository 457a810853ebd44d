"""ctypes binding of libcypress_b200.so (include/cypress_b200.h).  Marshalling only.

The shared library is built in-tree by ``paper_2504_07004_b200.build.build()``
(called from ``__graft_entry__.build()``).  There is no fallback: if the
library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcypress_b200.so")
_PRODUCT_PATH = LIB_PATH

# Every symbol include/cypress_b200.h declares (checked by tests/test_abi_cpu.py).
EXPORTS = (
    "cy_gemm", "cy_gemm_batched", "cy_dual_gemm", "cy_dual_gemm_glu", "cy_gemm_rowreduce", "cy_status_string",
    "cy_num_configs", "cy_config_info", "cy_force_config", "cy_last_config", "cy_launch_count",
    "cy_last_kernel_info", "cy_gemm_replicated", "cy_attention_fwd", "cy_peer_barrier", "cy_gemm_splitk",
    "cy_gemm_splitk_workspace_size", "cy_last_splits",
)

CY_OK = 0
STATUS_NAMES = {0: "CY_OK", 1: "CY_ERR_INVALID_VALUE", 2: "CY_ERR_MISALIGNED",
                3: "CY_ERR_UNSUPPORTED_DEVICE", 4: "CY_ERR_LAUNCH", 5: "CY_ERR_INTERNAL"}
CY_F16, CY_BF16 = 0, 1
CY_DUAL_PAIR, CY_DUAL_SUM = 0, 1
CY_ACT_SILU, CY_ACT_GELU_TANH = 0, 1


class CyError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{what}: {load().cy_status_string(status).decode()}")


_lib = None


def use_library(path: str) -> None:
    """Timing experiments only (scripts/): load an experiment build instead of the product library.
    Must run before the first call; tests, smoke() and bench.py never use it."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("library already loaded")
    LIB_PATH = path


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"cypress_b200: CUDA extension {LIB_PATH} is missing -- run `python -c "
            f"'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    i64, f32, vp, ci = ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_int
    lib.cy_gemm.argtypes = [ci, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, vp, i64, vp]
    if hasattr(lib, "cy_gemm_splitk"):
        lib.cy_gemm_splitk.argtypes = [ci, i64, i64, i64, i64, f32, vp, i64, i64, vp, i64, i64, f32, vp, i64, i64,
                                       vp, i64, i64, ci, vp, ctypes.c_size_t, vp]
        lib.cy_gemm_splitk.restype = ci
        lib.cy_gemm_splitk_workspace_size.argtypes = [ci, i64, i64, i64, i64, ci]
        lib.cy_gemm_splitk_workspace_size.restype = ctypes.c_size_t
        lib.cy_last_splits.restype = ci
    lib.cy_gemm_batched.argtypes = [ci, i64, i64, i64, i64, f32, vp, i64, i64, vp, i64, i64, f32,
                                    vp, i64, i64, vp, i64, i64, vp]
    lib.cy_dual_gemm.argtypes = [ci, ci, i64, i64, i64, f32, vp, i64, vp, i64, vp, i64, f32, vp, i64,
                                 vp, i64, vp, i64, vp, i64, vp]
    lib.cy_dual_gemm_glu.argtypes = [ci, ci, i64, i64, i64, f32, vp, i64, vp, i64, vp, i64, vp, i64, vp]
    lib.cy_gemm_replicated.argtypes = [ci, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64,
                                       ctypes.POINTER(ctypes.c_void_p), ci, i64, i64, i64, vp]
    lib.cy_attention_fwd.argtypes = [ci, i64, i64, i64, i64, i64, f32, ci, vp, vp, vp, vp, vp, vp]
    lib.cy_attention_fwd.restype = ci
    if LIB_PATH != _PRODUCT_PATH and not hasattr(lib, "cy_peer_barrier"):
        pass  # an older experiment build (scripts/): no peer barrier
    else:
        lib.cy_peer_barrier.argtypes = [ctypes.POINTER(ctypes.c_void_p), ci, ci, ctypes.c_uint32, vp]
        lib.cy_peer_barrier.restype = ci
    lib.cy_gemm_rowreduce.argtypes = [ci, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, vp, i64,
                                      vp, vp]
    for f in ("cy_gemm", "cy_gemm_batched", "cy_dual_gemm", "cy_dual_gemm_glu", "cy_gemm_rowreduce",
              "cy_gemm_replicated"):
        getattr(lib, f).restype = ci
    lib.cy_status_string.argtypes = [ci]
    lib.cy_status_string.restype = ctypes.c_char_p
    lib.cy_num_configs.restype = ci
    lib.cy_config_info.argtypes = [ci, ctypes.POINTER(ci), ctypes.POINTER(ci), ctypes.POINTER(ci),
                                   ctypes.POINTER(ci)]
    lib.cy_config_info.restype = ci
    lib.cy_force_config.argtypes = [ci]
    lib.cy_force_config.restype = ci
    lib.cy_last_config.restype = ci
    lib.cy_launch_count.restype = i64
    lib.cy_last_kernel_info.argtypes = [ctypes.POINTER(ci)] * 8
    lib.cy_last_kernel_info.restype = ci
    _lib = lib
    return lib


def check(status: int, what: str):
    if status != CY_OK:
        raise CyError(status, what)
