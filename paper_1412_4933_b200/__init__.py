"""pedflow-b200: B200-native per-time-step grid update of the bi-directional
pedestrian model of arXiv 1412.4933 (LEM and ACO), behind the reference
simulator's StepEngine API. See DESIGN.md."""
from .engine import (  # noqa: F401
    ConfigError,
    EngineOptions,
    ExecutorKind,
    Model,
    RunReport,
    ScenarioConfig,
    SimState,
    StateCorrupt,
    StepEngine,
    StepReport,
    StepSeriesRow,
    band_height,
    new_environment,
    run_scenario,
    validate,
)
from .ensemble import Ensemble  # noqa: F401

__version__ = "0.1.0"
