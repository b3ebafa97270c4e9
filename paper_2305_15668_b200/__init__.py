"""B200-native FedHC round hot path (arxiv 2305.15668), drop-in for `fedsim`.

Same public API as the reference package (fedsim/__init__.py:30-54); the
compute runs in libfedhc.so (hand-written sm_100a CUDA + a native C++ round
DES).  Importing this package loads libfedhc.so and fails loudly if it is
missing -- there is no CPU fallback.
"""

from . import _abi  # noqa: F401  (loads libfedhc.so or raises ImportError)
from .experiment import DataParams, DeviceFederation, ExperimentReport, TrainParams, run_experiment
from .planner import (CostCoefficients, Participant, ScheduleEntry, SchedulerState, maxmin_allocate, rate,
                      schedule_greedy, schedule_resource_aware, work_units)
from .roundsim import RoundReport, RoundSimulator, run_round
from .spec import (ClientProfile, DemandPhase, DistributionSpec, FleetConfig, WorkloadSpec, case_study_fleet,
                   generate_fleet, load_fleet, save_fleet)

__all__ = [
    "ClientProfile",
    "CostCoefficients",
    "DataParams",
    "DemandPhase",
    "DistributionSpec",
    "ExperimentReport",
    "FleetConfig",
    "Participant",
    "ScheduleEntry",
    "SchedulerState",
    "TrainParams",
    "WorkloadSpec",
    "case_study_fleet",
    "generate_fleet",
    "load_fleet",
    "maxmin_allocate",
    "rate",
    "run_experiment",
    "run_round",
    "save_fleet",
    "schedule_greedy",
    "schedule_resource_aware",
    "work_units",
    # B200-native additions
    "DeviceFederation",
    "RoundSimulator",
    "RoundReport",
]
