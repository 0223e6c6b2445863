"""B200-native (sm_100a) DICE expert-parallel MoE sampling path.

Drop-in for the reference simulator's model / policy / schedule API
(dicesim, /root/reference/pkg/src/dicesim) with the MoE layer math, token
exchange and staleness buffers on hand-written CUDA kernels.
"""
from .errors import (ConfigurationError, ContractError, NativeLibraryError,
                     NumericalDivergenceError, NumericsError, OracleScaleError,
                     SimulatorError)

__version__ = "0.1.0"
from .model import (ActivationBlock, ModelConfig, RouteDecision, ToyModel, combine_outputs,
                    denoise_update, expert_forward, gate, init_model, local_block, model_hash,
                    preset, routed_rows, sample_x0, shared_forward, splitmix64,
                    step_similarity, StepSimilarity)
from .policies import (NEUTRAL, CondStrategy, PolicyConfig, SyncStrategy, TokenCache,
                       apply_conditional, dice_policy, is_sync_step, random_keep_slots,
                       reduced_slots, select_sync_layers)
from .cluster import (ClusterConfig, Placement, build_placement, per_device_bytes,
                      plan_all_to_all)
from .schedules import (DeviceRunner, GpuTimeline, RunResult, StalenessRecord, Strategy,
                        run_sampling)
