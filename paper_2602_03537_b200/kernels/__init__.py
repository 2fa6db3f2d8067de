"""Backend identity (drop-in for nestquant.kernels, kernels/__init__.py:1-24).

There is exactly one backend: libmatq.so, hand-written CUDA for sm_100a.
No environment switch and no numpy fallback -- importing this package
without the built library raises ImportError.
"""

from .. import _lib

HAVE_COMPILED = True


def backend_name() -> str:
    return "cuda-sm%d" % _lib.lib().mq_arch()


def simd_kind() -> str:
    """Counterpart of _core.simd_kind() (_core.pyx:19-21)."""
    return "sm_%da" % _lib.lib().mq_arch()
