"""Configuration, enums, report and error types of the drop-in ``spgemm``.

Mirrors the reference's public surface so a ``sketchgemm`` user can switch:
``EngineConfig`` / ``WorkflowOverride`` / ``RunReport`` / exceptions
(``engine.py:39-110``), ``TierConfig`` / ``PlanKind`` (``accumulate.py:39-71``),
the workflow thresholds (``analysis.py:26-33``).  Added B200-only knobs are
keyword arguments with defaults that keep the reference behaviour.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

UPPER_BOUND_AVG_PRODUCTS = 64.0
ER_THRESHOLD = 8.0
CR_THRESHOLD = 8.0
REGISTER_ER_THRESHOLD = 48.0
DEFAULT_SAMPLE_RATIO = 0.03
DEFAULT_SAMPLE_MIN = 600
DEFAULT_SAMPLE_MAX = 10_000
HASH_LOAD_LIMIT = 0.8
PRECISION_FOR = {32: 5, 64: 6, 128: 7}


class ResourceLimitError(RuntimeError):
    """Staged output would exceed the configured memory budget (engine.py:39-40)."""


class DeadlineExceeded(RuntimeError):
    """Cooperative per-run timeout hit between pipeline stages (engine.py:43-44)."""


class CudaLibraryError(RuntimeError):
    """The sm_100a library is missing or a kernel launch failed."""


class WorkflowOverride(enum.Enum):
    AUTO = "auto"
    FORCE_SYMBOLIC = "symbolic"
    FORCE_ESTIMATE = "estimate"
    FORCE_UPPER_BOUND = "upper"


class WorkflowKind(enum.Enum):
    UPPER_BOUND = "upper"
    HLL_ESTIMATION = "estimate"
    SYMBOLIC = "symbolic"


class PlanKind(enum.IntEnum):
    HASH = 0
    ENHANCED_HASH = 1
    DENSE = 2
    ESC = 3
    FALLBACK = 4


@dataclass
class TierConfig:
    """Accumulator ladder (accumulate.py:47-71); same defaults and validation."""

    hash_capacities: tuple = (256, 512, 1024, 2048, 4096)
    enhanced_hash_capacity: int = 12288
    dense_spans: tuple = (1024, 2048, 4096, 8192, 16384)
    esc_max_products: int = 64
    expansion_coef: float = 1.5
    bitmap_query_threshold: float = 2.0

    def __post_init__(self):
        caps = list(self.hash_capacities)
        spans = list(self.dense_spans)
        if caps != sorted(caps) or spans != sorted(spans):
            raise ValueError("tier lists must be ascending")
        if any(c & (c - 1) for c in caps):
            raise ValueError("hash capacities must be powers of two")
        if self.expansion_coef < 1.0:
            raise ValueError("expansion_coef must be >= 1")
        if len(caps) > 8 or len(spans) > 8:
            raise ValueError("at most 8 hash capacities and 8 dense spans are supported")


@dataclass
class EngineConfig:
    """Reference fields (engine.py:54-74) plus B200 options.

    ``workers`` is accepted for API compatibility and ignored (the device
    decides its own parallelism; output never depends on it).  ``dtype`` picks
    the value type of the multiply ("f64" or "f32"; fp32 accumulates in fp64).
    ``return_device`` returns C as a ``DeviceCsr`` (torch CUDA tensors) instead
    of copying it to a host ``CsrMatrix``.
    """

    workflow: WorkflowOverride = WorkflowOverride.AUTO
    registers: int | None = None
    tiers: TierConfig = field(default_factory=TierConfig)
    coef: float | None = None
    sample_ratio: float = DEFAULT_SAMPLE_RATIO
    sample_min: int = DEFAULT_SAMPLE_MIN
    sample_max: int = DEFAULT_SAMPLE_MAX
    seed: int = 0
    workers: int = 1
    staging_limit_bytes: int | None = None
    compute_estimation_errors: bool = False
    # B200 options
    device: int | None = None
    dtype: str | None = None
    return_device: bool = False
    stream: object | None = None
    # fill RunReport.window_stats (row/product/nnz totals of the rows the
    # window kernel k_bmr processes; bench.py's roofline), a few reductions
    window_stats: bool = False
    # host results from the recycled pinned pool (device.HOST_POOL): repeated
    # calls download C by direct DMA with no page faults
    host_pool: bool = False
    # size hash-counted rows of the symbolic pass by products / conservative
    # CR; counts stay exact (overfull rows are recounted)
    assisted_symbolic: bool = True
    # symbolic workflow: rows of <= 1024 products skip the count pass and are
    # accumulated once into a product-sized staging slab, then compacted
    stage_short_rows: bool = True
    # multi-GPU: the workflow decision of the WHOLE product, made once on the
    # root rank (shard.Decision); a shard then skips its own sampling and
    # reports the global er / cr_hat / workflow / registers
    decision: object | None = None
    # values summed in the reference's sequential stream order after the
    # structure is final (sg_det_values): bit-identical run to run, as the
    # reference guarantees (engine.py:13-14); refbind turns it on
    deterministic: bool = False

    def __post_init__(self):
        if self.registers is not None and self.registers not in PRECISION_FOR:
            raise ValueError(f"registers must be one of {sorted(PRECISION_FOR)}")
        if self.sample_ratio <= 0 or self.sample_min <= 0 or self.sample_max <= 0:
            raise ValueError("sampling parameters must be positive")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.dtype not in (None, "f64", "f32"):
            raise ValueError("dtype must be 'f64' or 'f32'")


@dataclass
class RunReport:
    """Same fields as the reference report (engine.py:91-110) plus device extras."""

    workflow: str
    registers: int
    er: float
    cr_hat: float | None
    cr_true: float | None
    analysis_ms: float
    sketch_ms: float
    predict_ms: float
    numeric_ms: float
    fallback_ms: float
    compact_ms: float
    total_ms: float
    overflow_row_count: int
    nnz_c: int
    total_products: int
    bitmap_query: bool
    est_mean_rel_err: float | None = None
    est_std_rel_err: float | None = None
    # device extras
    gflops: float | None = None
    kernel_ms: dict | None = None
    n_gpus: int = 1
    window_stats: dict | None = None


def select_registers(er: float) -> int:
    """analysis.py:199-203"""
    if er < 0:
        raise ValueError("ER must be non-negative")
    return 32 if er < REGISTER_ER_THRESHOLD else 64


def select_workflow(avg_products: float, er: float, cr_hat: float) -> WorkflowKind:
    """analysis.py:206-217"""
    if avg_products < UPPER_BOUND_AVG_PRODUCTS:
        return WorkflowKind.UPPER_BOUND
    if er >= ER_THRESHOLD and cr_hat >= CR_THRESHOLD:
        return WorkflowKind.HLL_ESTIMATION
    return WorkflowKind.SYMBOLIC


def cr_variance_bound(cv: float, m: int, n_sampled: int) -> float:
    """Relative variance of 1/CR for the sampled estimator (analysis.py:220-229)."""
    if n_sampled <= 0:
        raise ValueError("n_sampled must be positive")
    eps2 = (1.04 / m ** 0.5) ** 2
    return (eps2 + cv * cv * (1.0 + eps2)) / n_sampled
