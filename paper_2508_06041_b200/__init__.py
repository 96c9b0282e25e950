"""B200-native DP-LLM decode hot path (drop-in for the reference ``dpq`` runtime).

Per-linear-layer precision selection fused with an any-precision bitplane
GEMV, written as hand-tuned sm_100a CUDA behind a C-ABI (libdpq_b200.so,
include/dpq_b200.h). The public surface mirrors the reference's
``dpq/__init__.py:8-23`` for the decode path: model/store/plan types and file
formats, ``select_precision``, ``DecodeEngine``, ``decode`` and
``eval_perplexity``. Offline planning (allocator, fitter, sensitivity) is out
of scope; plans built by the reference load unchanged.
"""

from .model import (KINDS, LayerId, ModelConfig, ModelWeights, init_model, export_weights, forward, backward,
                    teacher_forced_loss,
                    load_weights, layer_ids, layer_shape)
from .quant import (QuantizedLayer, BitPlaneStore, QuantError, quantize_layer, dequantize,
                    delta_weights, gemv, quantize_model, save_store, load_store, load_device_store, file_hash,
                    pack_codes, unpack_codes)
from .estimator import (ErrorEstimator, LinearEstimator, ProjectionEstimator, ExactEstimator,
                        IMMEDIATE, PREVIOUS_RESIDUAL, exact_error, resolve_input_source,
                        translate_threshold, collect_error_samples, build_projection, calibrate_projection)
from .runtime import (PrecisionPlan, PlanLayer, DecodeEngine, DecodeTrace, StepRecord,
                      ProvenanceError, decode, eval_perplexity, qos_stats, save_plan, load_plan,
                      sentinel_static_plan, select_precision, incurred_error_comparison)

__version__ = "0.1.0"
