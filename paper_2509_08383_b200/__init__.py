"""B200-native CutMax decoding core (arXiv 2509.08383): batched CutMax argmax and
the Beta-cut nucleus sampler as hand-written sm_100a CUDA kernels behind a C ABI
(include/pam_c_api.h) and the reference's `polyargmax` interface."""
from . import _abi
from .errors import (CudaError, DegenerateInputError, DomainError, Error, FormatError, InvalidParamsError,
                     NonFiniteError, RangeError, SingularityError, TieWarning)
from .polyargmax import (ApproxConfig, CutMaxParams, ResidualStats, SampleOutcome, SamplerConfig, ScoreVector,
                         betaInverseCdf, cutmax, cutmax_batch, cutmax_batch_device, cutmaxStep, goldschmidtInv,
                         goldschmidtInvSqrt, gumbel_sample_batch_device, gumbelFromUniform, gumbelMaxSample,
                         kernel_launch_count, launch_info, nucleus_sample_batch_device, nucleusAlpha,
                         nucleusOneShotSample, uniform, violationExperiment, ingest, ingest_pinned, write_lgt1,
                         convergence_trace_batch_device, convergenceTrace, cutmax_jvp_batch_device, cutmaxJvp,
                         cutmaxJacobian, geometry_override, general_p3_kernel, nucleus_set_batch_device, nucleusSet)

__all__ = [
    "ApproxConfig", "CutMaxParams", "ResidualStats", "SampleOutcome", "SamplerConfig", "ScoreVector",
    "betaInverseCdf", "cutmax", "cutmax_batch", "cutmax_batch_device", "cutmaxStep", "goldschmidtInv",
    "goldschmidtInvSqrt", "gumbel_sample_batch_device", "gumbelFromUniform", "gumbelMaxSample",
    "kernel_launch_count", "launch_info", "nucleus_sample_batch_device", "nucleusAlpha", "nucleusOneShotSample",
    "uniform", "violationExperiment", "ingest", "ingest_pinned", "write_lgt1", "convergence_trace_batch_device", "convergenceTrace",
    "cutmax_jvp_batch_device", "cutmaxJvp", "cutmaxJacobian", "Error", "FormatError", "SingularityError", "DegenerateInputError", "InvalidParamsError", "RangeError", "DomainError",
    "NonFiniteError", "CudaError", "TieWarning", "geometry_override", "general_p3_kernel", "nucleus_set_batch_device", "nucleusSet",
]
