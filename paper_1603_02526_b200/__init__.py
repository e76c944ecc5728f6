"""B200-native factor-graph ADMM (parADMM, arXiv:1603.02526).

Drop-in for the reference package ``fgadmm``: same graph, operator,
problem and engine API; the five-phase iteration runs as hand-written
sm_100a kernels in ``libfgadmm_b200.so`` (C-ABI: include/fgadmm_b200.h).
"""

from .engine import (
    METRICS_HEADER,
    PHASES,
    AdmmState,
    DevicePlan,
    RunConfig,
    RunReport,
    device_plan,
    init_state,
    iterate,
    pinned_state,
    residuals,
    run,
    update_m,
    update_n,
    update_u,
    update_x,
    update_z,
)
from .graph import (DOCUMENT_VERSION, Edge, FactorGraph, FunctionNode, GraphBuilder,
                    VariableNode, deserialize, serialize)
from .operators import (
    Collision,
    Equality,
    HalfPlane,
    LabeledPoint,
    LinearSystem,
    MpcCost,
    MpcDyn,
    MpcInit,
    NanTest,
    Quadratic,
    Radius,
    SvmMargin,
    SvmNorm,
    SvmSlack,
    Wall,
    collision_prox,
    equality_prox,
    mpc_cost_prox,
    mpc_dyn_prox,
    mpc_init_prox,
    radius_prox,
    svm_margin_prox,
    svm_norm_prox,
    svm_slack_prox,
    wall_prox,
)
from .problems import (
    MpcSpec,
    PackingSpec,
    SvmSpec,
    build_mpc,
    build_packing,
    build_svm,
    gen_gaussian_arrays,
    gen_gaussian_data,
    load_points,
    mpc_qp_solution,
    packing_init,
    pendulum_linearization,
    save_points,
    svm_accuracy,
    svm_objective,
    svm_qp_solution,
    unit_triangle,
)
from .prox import ProxFactor, check_prox_input, operator_class, register, registered_kinds

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
