"""ctypes binding of libmatq.so (include/matq.h).

The package has no CPU fallback: importing this module fails loudly when the
CUDA library has not been built, and every call checks the C status.  The
binding is the Python counterpart of the reference's Cython bridge
(kernels/_core.pyx:8-16), which binds packed_kernels.h the same way.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# MQ_LIB_PATH: load an alternative build (tuning experiments only)
LIB_PATH = os.environ.get("MQ_LIB_PATH") or os.path.join(HERE, "libmatq.so")

MQ_OK = 0
MQ_ERR_INVALID = 1
MQ_ERR_CODE_RANGE = 2
MQ_ERR_WORKSPACE = 3
MQ_ERR_CUDA = 4

MQ_CHILD = 1
MQ_X_F32 = 2
MQ_Y_F32 = 4
MQ_PDL = 8

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "libmatq.so is not built (%s); run `python -c \"import __graft_entry__ as g; g.build()\"` "
        "-- there is no CPU fallback" % LIB_PATH)

_L = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_sz = ctypes.c_size_t
_f = ctypes.c_float

_SIGS = {
    "mq_arch": ([], _i),
    "mq_version": ([], ctypes.c_char_p),
    "mq_last_error": ([], ctypes.c_char_p),
    "mq_layout_dims": ([_i, _i, _i, _vp, _vp, _vp], _i),
    "mq_blob_bytes": ([_i, _i, _i, _i], _sz),
    "mq_tscales_bytes": ([_i, _i, _i], _sz),
    "mq_pack_blob": ([_vp, _ll, _i, _i, _i, _vp, _i, _vp, _vp, _vp], _i),
    "mq_slice": ([_vp, _i, _i, _i, _i, _i, _vp, _ll, _vp], _i),
    "mq_dequant": ([_vp, _vp, _i, _i, _i, _i, _i, _f, _vp, _vp, _ll, _vp], _i),
    "mq_materialize_child": ([_vp, _i, _i, _i, _i, _vp, _vp], _i),
    "mq_gemv_workspace_bytes": ([_i, _i, _i, _i], _sz),
    "mq_gemv": ([_vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _f, _i, _vp, _sz, _vp], _i),
    "mq_gemm_workspace_bytes": ([_i, _i, _i, _i], _sz),
    "mq_gemm": ([_vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _f, _i, _vp, _sz, _vp], _i),
    "mq_stack_plan_bytes": ([], _sz),
    "mq_stack_table_bytes": ([_i], _sz),
    "mq_stack_plan": ([_vp, _i, _i, _i, _i, _vp, _vp, _vp], _i),
    "mq_stack_run": ([_vp, _vp, _vp, _sz, _vp], _i),
    "mq_stack_epoch": ([_vp, _vp, _sz, _vp, _i, _vp], _i),
    "mq_slice_elementwise": ([_vp, _ll, _i, _i, _i, _vp, _vp, _vp], _i),
    "mq_dequant_f64": ([_vp, _i, _i, _vp, _i, _i, _i, _i, _vp, _vp, _vp], _i),
    "mq_dequant_value_f64": ([_vp, _vp, _ll, _i, _i, _vp, _vp, _vp], _i),
    "mq_matmul_ref": ([_vp, _i, _i, _vp, _i, _vp, _vp], _i),
    "mq_pack_ref_layout": ([_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp], _i),
    "mq_unpack_ref_layout": ([_vp, _vp, _vp, _i, _i, _vp, _vp], _i),
    "mq_select_codes": ([_vp, _ll, _i, _i, _vp, _i, _i, _vp, _vp, _i, _vp, _ll, _vp], _i),
    "mq_rtn_f64": ([_vp, _vp, _ll, _i, _vp, _vp, _vp], _i),
    "mq_round_half_away_f64": ([_vp, _ll, _vp, _vp], _i),
    "mq_fit_grid": ([_vp, _ll, _i, _i, _i, _vp, _vp, _i, _vp, _i, _vp, _vp], _i),
    "mq_add_rmsnorm": ([_vp, _vp, _vp, _vp, _i, _i, _f, _vp], _i),
    "mq_rope_kv": ([_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp], _i),
    "mq_qknorm_rope_kv": ([_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _f, _vp], _i),
    "mq_silu_mul": ([_vp, _vp, _i, _i, _vp], _i),
    "mq_attn_decode": ([_vp, _vp, _vp, _vp, _vp, _f, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp], _i),
    "mq_gptq_block": ([_vp, _ll, _i, _i, _i, _i, _vp, _i, _i, _vp, _ll, _vp, _vp, _i, _vp, _ll, _vp, _ll, _vp,
                       _ll, _vp], _i),
}

EXPORTS = tuple(_SIGS)

for _name, (_args, _res) in _SIGS.items():
    if os.environ.get("MQ_LIB_PATH") and not hasattr(_L, _name):
        continue  # an older tuning build (MQ_LIB_PATH) may predate an entry point
    _fn = getattr(_L, _name)
    _fn.argtypes = _args
    _fn.restype = _res


class StackLayer(ctypes.Structure):
    """struct mq_stack_layer (include/matq.h)."""

    _fields_ = [("blob", ctypes.c_void_p), ("X", ctypes.c_void_p), ("Y", ctypes.c_void_p),
                ("ldx", ctypes.c_int), ("ldy", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
                ("out_scale", ctypes.c_float), ("r", ctypes.c_int),
                ("xop", ctypes.c_int), ("res_in", ctypes.c_void_p), ("res_out", ctypes.c_void_p),
                ("norm_w", ctypes.c_void_p), ("ldres", ctypes.c_int), ("eps", ctypes.c_float),
                ("yop", ctypes.c_int)]


MQ_XOP_NONE, MQ_XOP_ADD_RMSNORM, MQ_XOP_SILU_MUL = 0, 1, 2
MQ_YOP_NONE, MQ_YOP_SILU_PAIRS = 0, 1


class MatqError(RuntimeError):
    """A libmatq call failed; .status holds the MQ_ERR_* code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def last_error() -> str:
    return (_L.mq_last_error() or b"").decode()


def call(name: str, *args) -> None:
    st = getattr(_L, name)(*args)
    if st != MQ_OK:
        raise MatqError(st, "%s failed (status %d): %s" % (name, st, last_error()))


def lib():
    return _L


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("matq needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_ERR_SCRATCH: dict[int, torch.Tensor] = {}


def err_scratch() -> torch.Tensor:
    dev = torch.cuda.current_device()
    t = _ERR_SCRATCH.get(dev)
    if t is None:
        t = torch.zeros(1, dtype=torch.int32, device="cuda")
        _ERR_SCRATCH[dev] = t
    return t
