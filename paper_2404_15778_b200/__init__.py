"""B200-native BASS (batched attention-optimized speculative sampling).

Drop-in for the reference package's decode API (`batchspec`,
ref:__init__.py:8-84, hot-path subset): the same request/result types,
controllers and providers protocol, with the hot path in libbass.so
(hand-written sm_100a CUDA behind the C ABI of include/bass.h).
"""

from .attention import AttentionStrategy, attend_device
from .control import (AdaptiveDraftController, DraftLengthParams, DraftLengthState,
                      FixedDraftController, init_state, update)
from .engine import (CudaEngine, GenerationRequest, GenerationResult, SpecStepOutcome,
                     decode_regular, decode_speculative, step_trace)
from .model import (CudaAlignedDraft, CudaContext, CudaModel, DeviceWeights, ModelConfig,
                    desk_config)
from .quant import GroupAxis, QuantTensor, int_gemm_dequant
from .sampling import (ROLE_DRAFT, ROLE_VERIFY, device_accept, device_shape_sample,
                       device_uniforms)

__version__ = "0.1.0"
