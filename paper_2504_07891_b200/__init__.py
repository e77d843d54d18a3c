"""B200-native SpecReason inner loop (arXiv 2504.07891).

Drop-in for the reference ``stepspec`` hot path: the same plugin API
(``Backend``, request/result types, ``extract_score``), the same driver
(``run_trajectory``, ``run_vanilla``, ``segment_step``, ...), and a
``B200Backend`` whose generation and scoring run as hand-written sm_100a
kernels behind the C-ABI declared in ``include/specreason_b200.h``.
"""

from .contract import (
    Backend,
    BackendError,
    BackendMisbehavior,
    FinishReason,
    GenerationRequest,
    GenerationResult,
    ScoreParseFailure,
    TransportError,
    VerificationRequest,
    count_new_prompt_tokens,
    extract_score,
)
from .domain import (
    END_THINK_MARKER,
    THINK_OPEN_MARKER,
    AcceptanceThreshold,
    BackendProfile,
    BackendRole,
    Decision,
    EngineConfig,
    LatencyBreakdown,
    Phase,
    ReasoningStep,
    RunMetrics,
    Scheme,
    StepProducer,
    TrajectoryState,
    UtilityScore,
    decide_acceptance,
    total_latency,
)
from .driver import (
    StepAction,
    StepOutcome,
    TrajectoryResult,
    force_first_n,
    run_trajectory,
    run_vanilla,
    segment_step,
    validate_trajectory,
)
from .pricing import trajectory_seed

__version__ = "0.1.0"


def __getattr__(name: str):
    # the device backend pulls in torch + the native library lazily
    if name in ("B200Backend", "build_pair"):
        from . import backend

        return getattr(backend, name)
    raise AttributeError(name)
