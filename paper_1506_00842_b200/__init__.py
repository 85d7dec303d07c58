"""paper_1506_00842_b200 — B200-native core of Falch & Elster's ML auto-tuner
(arXiv 1506.00842), a drop-in for the reference package `mltune`'s hot path.

The public names mirror `mltune` (/root/reference/pkg/src/mltune/__init__.py):
spaces, measurement records, the ensemble model, and the tuner. The numeric
work — index decode/encode, validity masks, full-space ensemble prediction
with top-M selection, and ensemble training — runs in hand-written sm_100a
CUDA (libmltune_b200.so, C ABI in include/mltune_b200.h). There is no CPU
fallback: without the library or a B200 the numeric calls raise.
"""

from .errors import (AllCandidatesInvalidError, ConfigMismatchError, DivergenceError, EmptySpaceError,
                     InsufficientDataError, InvalidConfigurationError, MltuneError, NativeUnavailableError,
                     ParseError, RunnerError)
from .space import (BUILTIN_SPACE_NAMES, Configuration, ParamDef, ParamSpace, ValidityRule, builtin_space,
                    load_space, save_space, space_from_json, space_to_json)
from .measurement import Outcome, Sample, SampleSet
from .model import (Encoder, Ensemble, Network, TrainConfig, forward, gradient, load_model, model_from_json,
                    predict, save_model, train_ensemble, train_network)
from .tuner import (TunerConfig, TuningReport, autotune, exhaustive_search, measure_configs, top_m_arrays,
                    top_m_predicted)
from .surrogate import B200SurrogateRunner
from .install import install, uninstall

__version__ = "0.1.0"
