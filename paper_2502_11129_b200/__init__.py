"""paper_2502_11129_b200 — B200-native batched variant simulation.

The hot path of arXiv 2502.11129's reference (`hetbench`): evaluating
thousands of independent robot variants through many physics steps, as one
persistent sm_100a kernel per batch behind the reference's batch_executor
contract.  Native code: libhbgpu.so (csrc/, C ABI in include/hbgpu.h).
"""
from .executor import (ALL_MODELS, BatchExecutor, BatchFailure, BatchRequest, BatchResult,
                       DeviceContext, GpuExecutor, ModelKind, MultiGpuExecutor, NumericalBlowup,
                       RESULT_DTYPE, body_count, build_states, constraint_count, device_count,
                       format_blowup, kernel_name, parse_model_kind, pinned_seeds, state_rows,
                       to_string,
                       validate_request)
from .scheduler import (AllocationPlan, CalibrationProfile, HybridResult, calibrate, calibrate_n,
                        format_plan, naive_sum, plan_allocation, plan_allocation_n,
                        plan_allocation_optimal, run_hybrid, run_sharded, ShardedResult,
                        snap_equal_times)
from .ea import (EaResult, PhaseProfile, Population, report_profile, rng_at, run_ea,
                 run_ea_native, stable_order_desc)

from .monitor import GpuUtilSampler, KneeRegime, Stats, detect_saturation_knee, summarize

LIB_PATH = __import__("paper_2502_11129_b200._lib", fromlist=["LIB_PATH"]).LIB_PATH

__all__ = [n for n in dir() if not n.startswith("_")]
