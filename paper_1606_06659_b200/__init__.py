"""B200-native slice-within-Gibbs sweep for the two-level Poisson-lognormal
RNA-seq model (arXiv 1606.06659), behind the reference countmc engine API.

The compute path is ``lib/libcountmc_b200.so`` (CUDA, sm_100a) reached through
the C-ABI in ``include/countmc_b200.h``; this package mirrors the reference's
``GibbsEngine`` interface on top of it.
"""
from .engine import (ChainOutput, ChainState, ConfigError, ContrastSpec, Diagnostics,
                     ContrastTerm, CountMatrix, DeviceError, GibbsEngine,
                     LoadError, LoopbackGroup, ModelSpec, Moments, NormalizationError, ParamRef,
                     PriorConfig, RunConfig, estimate_offsets, load_counts,
                     DesignTable, load_model_matrix, load_offsets,
                     SamplerStallError, SimSpec, SliceConfig, TuningState,
                     builtin_design, disjunction_combine, generate,
                     heterosis_contrast, parse_param_ref)
from ._abi import load_library, sizes

__all__ = [
    "ChainOutput", "ChainState", "ConfigError", "ContrastSpec", "ContrastTerm", "Diagnostics",
    "CountMatrix", "DeviceError", "GibbsEngine", "LoadError", "LoopbackGroup", "ModelSpec",
    "Moments",
    "NormalizationError", "estimate_offsets", "load_counts",
    "DesignTable", "load_model_matrix", "load_offsets",
    "ParamRef", "PriorConfig", "RunConfig", "SamplerStallError", "SimSpec",
    "SliceConfig", "TuningState", "builtin_design", "disjunction_combine",
    "generate", "heterosis_contrast", "parse_param_ref", "load_library", "sizes",
]
