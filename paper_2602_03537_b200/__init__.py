"""B200-native sliced weight-only linear (MatGPTQ inference hot path).

Drop-in for the hot-path surface of the reference package ``nestquant``
(/root/reference/pkg/src/nestquant/__init__.py:10-34): slicing, grid
dequantisation, the child packing format, the packed matmul and the MatGPTQ
quantiser's searches (gptq, fit_grid), plus the
device-resident parent planes (``PlaneTensor``) and a torch module
(``MatLinear``).  All compute goes through libmatq.so (sm_100a CUDA behind a
C ABI, include/matq.h); there is no CPU fallback.
"""

from . import _lib  # noqa: F401  (fails loudly if libmatq.so is missing)
from .device import PlaneTensor, StackProgram, algorithmic_bytes, reserve_workspace
from .checkpoint import Checkpoint, CheckpointError, SlicedModel, read_checkpoint, write_checkpoint
from .config import mutate_level_switch
from .grid import (BitWidthSet, GridError, QuantGrid, base_scale, dequant, dequant_value, fit_grid, round_half_away,
                   rtn)
from .gptq import (CalibBatch, HessianFactor, QuantizeError, build_hessian, factor_inverse, quantize_layer,
                   select_codes)
from .matmul import (MatmulError, MatmulTask, PackedLayer, bench, matmul_packed,
                     matmul_packed_device, matmul_ref, random_task)
from .module import MatLinear
from .packing import PackedTensor, PackError, pack, pack_slice, to_canonical, to_interleaved, unpack
from .slicing import (BitConfig, NestedLayer, SlicedLayer, SliceError, slice_code, slice_layer,
                      slice_model, slice_to_code)

__version__ = "0.1.0"
