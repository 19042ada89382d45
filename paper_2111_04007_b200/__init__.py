"""paper_2111_04007_b200 (vpipe): a B200-native Varuna pipeline-parallel
training executor behind spotpipe's public API (sp/__init__.py:4-59).

Control plane (native C++ in libvpipe.so): the Varuna micro-batch schedule,
CutPoint identification / stage assignment, placement, micro-batch
accounting, the replica event kernel and the bubble predictor.
Data plane (sm_100a CUDA in libvpipe.so, driven from ``runtime``): per-stage
GPT-2 forward / recompute / backward, NVLink P2P between stages, NCCL DP
allreduce fused with unscale + overflow + Adam. ``Varuna``/``CutPoint`` are
imported lazily (they need torch).
"""

from .core import (  # noqa: F401
    ClusterState, ConfigError, HardwareSpec, InfeasibleError, JobSpec, ModelSpec,
    ParallelConfig, VM, make_block_model, uniform_cluster, uniform_stage_map, validate_config,
    B200_NVL8,
)
from .calibration import (  # noqa: F401
    CalibrationProfile, CutpointTimes, load_profile, ring_allreduce_seconds, save_profile,
    synthesize_profile, uniform_profile,
)
from .partitioner import (  # noqa: F401
    MemoryReport, OpProfile, Operation, StageAssignment, assign_stages, identify_cutpoints,
    load_op_profile, memory_check,
)
from .scheduler import (  # noqa: F401
    POLICY_GPIPE, POLICY_VARUNA, Schedule, Task, generate_gpipe_schedule,
    generate_varuna_schedule, makespan_us, schedule_from_csv, schedule_to_csv,
    validate_schedule,
)
from .simulator import Placement, SimulationResult, build_placement, simulate_minibatch  # noqa: F401
from .planner import PlanResult, micro_batches_for, plan, select_microbatch  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    if name in ("Varuna", "CutPoint", "StepResult", "LossScaler", "morph", "replan"):
        from . import runtime
        return getattr(runtime, name)
    if name in ("GPT2", "TransformerLayer"):
        from . import modules
        return getattr(modules, name)
    raise AttributeError(name)
