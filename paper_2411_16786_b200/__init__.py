"""B200-native (sm_100a) DICE expert-parallel MoE sampling path.

Drop-in for the reference simulator's model / policy / schedule API
(dicesim, /root/reference/pkg/src/dicesim) with the MoE layer math, token
exchange and staleness buffers on hand-written CUDA kernels.
"""
from .errors import (ConfigurationError, ContractError, NativeLibraryError,
                     NumericalDivergenceError, NumericsError, OracleScaleError,
                     SimulatorError)

__version__ = "0.1.0"
