"""B200-native asynchronous-Parareal hot path.

Drop-in for the hot path of the reference package ``pintlab``
(arXiv 2110.10762): the propagator plugin layer (``PROPAGATOR_RULES``,
``.apply``), the synchronous driver (``run_parareal`` and its helpers) and the
asynchronous driver (``run_async_parareal``), with every state in HBM and
every operation on hand-written sm_100a kernels (libpint_b200.so, C ABI in
include/pint_abi.h). There is no CPU fallback.
"""
from .async_engine import (
    POLICIES,
    POLICY_ADVERSARIAL,
    POLICY_RANDOM_FAIR,
    POLICY_ROUND_ROBIN,
    AsyncMapping,
    AsyncSchedule,
    AsyncTrace,
    EngineView,
    ScheduleValidation,
    UpdateRecord,
    update_counts,
    validate_schedule,
)
from .async_parareal import (
    FRESH_SLOT,
    REMEMBERED_SLOT,
    async_parareal_mapping,
    async_stop_check,
    simulate_async,
    run_async_parareal,
    simulate_parareal_async,
    run_async_parareal_device,
    audit_device_trace,
    DeviceAsyncResult,
)
from .errors import (
    ConfigError,
    ConvergenceFailure,
    DegenerateProblemError,
    DimensionError,
    HorizonExhausted,
    InvalidWeightError,
    NativeLibraryError,
    SingularMatrixError,
    SingularSystemError,
    InvalidThetaError,
    UndefinedLimitError,
    UnfittableError,
)
from .contraction import (
    CheckResult,
    ContractionReport,
    NormKind,
    RateComparison,
    async_convergence_check,
    compare_factors,
    contraction_factors,
    factors_from_norms,
    sync_convergence_check,
)
from .costmodel import (
    CostParams,
    SpeedupReport,
    async_cost,
    asymptotic_speedups,
    fit_overhead,
    measure_costs,
    model_report,
    sequential_cost,
    speedup_bound,
    sync_cost,
)
from .async_mp import run_async_parareal_mp
from .linalg import BlockVector
from .model import (
    PROPAGATOR_RULES,
    GPUPropagator,
    HeatIVP,
    LinearIVP,
    TimeDecomposition,
    backward_euler_propagator,
    forward_euler_propagator,
    heat1d_system,
    heat2d_system,
    heat3d_system,
    scalar_decay_system,
    trapezoidal_propagator,
)
from .parareal import (
    STOP_EXACT,
    STOP_KMAX,
    STOP_THRESHOLD,
    SyncEngine,
    SyncTrace,
    coarse_init,
    parareal_iterate,
    parareal_update,
    run_parareal,
    sequential_fine_solve,
)

__version__ = "0.1.0"
