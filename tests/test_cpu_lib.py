"""CPU-only checks of the native boundary and the host-side logic."""

import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "matq.h")).read()
    return sorted(set(re.findall(r"MQ_API\s+[\w\s\*]+?\b(mq_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2602_03537_b200 import _lib

    syms = _header_symbols()
    assert len(syms) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(mq_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # and the ctypes binding declares the same set
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a():
    from paper_2602_03537_b200 import _lib, kernels

    assert _lib.lib().mq_arch() == 100
    assert kernels.backend_name() == "cuda-sm100"
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_layout_queries():
    import ctypes

    from paper_2602_03537_b200 import _lib

    L = _lib.lib()
    Np, Kp, ngp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert L.mq_layout_dims(40, 600, 128, ctypes.byref(Np), ctypes.byref(Kp), ctypes.byref(ngp)) == 0
    assert (Np.value, Kp.value, ngp.value) == (48, 768, 6)
    # blob = planes + one fp32 scale per (row, group) embedded per step (G = 128)
    assert L.mq_blob_bytes(4096, 4096, 128, 8) == 4096 * 4096 + 4096 * 32 * 4
    assert L.mq_blob_bytes(4096, 4096, 128, 3) == 3 * 4096 * 4096 // 8 + 4096 * 32 * 4
    assert L.mq_blob_bytes(4096, 4096, 96, 8) == 4096 * 4096  # no embedded scales
    assert L.mq_tscales_bytes(4096, 4096, 128) == 4096 * 32 * 4
    assert L.mq_layout_dims(0, 10, 128, None, None, None) == _lib.MQ_ERR_INVALID
    # workspace query is host-only
    assert L.mq_gemv_workspace_bytes(16, 256, 1, 0) == 0  # one K step: no split-K
    assert L.mq_gemv_workspace_bytes(4096, 4096, 1, 0) % 4 == 0
    assert L.mq_gemv_workspace_bytes(4096, 4096, 33, 0) == 0  # above the GEMV limit


def test_invalid_arguments_fail_before_cuda():
    from paper_2602_03537_b200 import _lib

    L = _lib.lib()
    # unsupported bits / group size are rejected by validation, no device touched
    st = L.mq_gemv(1, 1, 1, 64, 1, 64, 1, 64, 64, 128, 8, 5, 1.0, 0, None, 0, None)
    assert st == _lib.MQ_ERR_INVALID and "unsupported bits" in _lib.last_error()
    st = L.mq_gemv(1, 1, 1, 64, 1, 64, 1, 64, 64, 48, 8, 4, 1.0, 0, None, 0, None)
    assert st == _lib.MQ_ERR_INVALID and "multiple of 32" in _lib.last_error()
    st = L.mq_slice_elementwise(None, 0, 3, 4, 0, None, None, None)
    assert st == _lib.MQ_ERR_INVALID and "cannot slice 4 bits out of 3" in _lib.last_error()


def test_host_emulation_of_device_decode(tmp_path):
    """K1 pack + K3 register decode, compiled for the host, vs the reference slice."""
    exe = str(tmp_path / "layout_emu")
    subprocess.run(["nvcc", "-std=c++17", "-O2", "--expt-relaxed-constexpr",
                    "-Wno-deprecated-gpu-targets", "-o", exe,
                    os.path.join(ROOT, "tests", "emu", "layout_emu.cu")], check=True)
    for n, k in ((40, 600), (17, 300), (16, 256), (1, 1)):
        res = subprocess.run([exe, str(n), str(k)], capture_output=True, text=True)
        assert res.returncode == 0, res.stdout
        assert res.stdout.startswith("OK")


def test_reference_api_validation_messages():
    from paper_2602_03537_b200 import BitConfig, SliceError, BitWidthSet, GridError, QuantGrid
    from paper_2602_03537_b200.slicing import _check_slice_args

    with pytest.raises(SliceError, match="cannot slice 4 bits out of 3"):
        _check_slice_args(3, 4)
    with pytest.raises(SliceError, match=">= 2"):
        _check_slice_args(8, 1)
    with pytest.raises(SliceError):
        BitConfig({"a": 5})
    assert BitConfig({"a": 2, "b": 4}, budget_bits=60).total_bits({"a": 10, "b": 10}) == 60
    with pytest.raises(GridError, match="distinct and sorted"):
        BitWidthSet((4, 3), (1.0, 1.0))
    with pytest.raises(GridError, match="scale floor"):
        QuantGrid(8, 128, np.zeros((2, 1), np.float32))
