"""B200-native (sm_100a) drop-in for the VLCache cache-reuse prefill path.

Same public names as the reference package `kvreuse` (__init__.py:3-16) for the
hot path: the encoder / KV cache store, the layer-wise recompute-budget
allocator and `prefill_with_reuse`.  Compute runs in libvlcache.so (hand-written
tcgen05 / TMA kernels) through a C ABI; there is no CPU fallback.
"""
from .config import ModelConfig
from .engine import (DecodeResult, FlopsBreakdown, ReuseMetrics, ReuseRequest, ReuseResult, apply_rope, count_flops,
                     decode_with_merged_kv, encode_image, forward_injected, plan_to_use_cached,
                     fill_store, fill_store_request, flops_from_masks, generate, prefill_batch_with_reuse, prefill_full,
                     prefill_with_reuse)
from .exceptions import (ConfigError, InputError, IntegrityError, KVReuseError, ParseError, PlanError,
                         SetupError, StaleCacheError)
from .model import KVTensors, ToyVLM, init_model, load_model, save_weights, weight_checksum
from .planner import BudgetSpec, objective, plan_bruteforce, plan_greedy, plan_static
from .plans import (ComputationMask, RecomputePlan, build_masks, load_plan, mean_ratio, recompute_count,
                    save_plan, validate_plan)
from .sensitivity import ProxySample, SensitivityTable, profile
from .sequence import Segment, TokenSequence, make_sequence
from .store import CacheStore, EncoderCacheEntry, ImageHash, KVCacheEntry, hash_image, hash_request

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"
