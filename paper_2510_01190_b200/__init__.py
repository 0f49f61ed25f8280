"""B200-native divergence-uncertainty hot path (arxiv 2510.01190), drop-in for ``divuq``.

The public names mirror the reference package's hot-path API
(/root/reference/pkg/src/divuq/__init__.py:9-96): ``fit_gaussian``,
``propagate_divergence``, ``divergence_deterministic``,
``stencil_distribution``, ``mc_divergence``, ``error_metrics`` and the data
types, plus the probability maps the reference keeps private
(``tail_probs`` / ``source_probability`` / ``sink_probability``), 3D twins,
and the fused ensemble pipeline.  ``device`` holds the torch-tensor
(HBM-resident) API, ``shard`` the z-slab multi-GPU driver.

Importing raises if the sm_100a library (libdivuq_b200.so) is missing --
there is no CPU fallback.
"""

from . import _lib  # noqa: F401  (fails loudly without the CUDA library)
from . import io  # noqa: F401  (DIVUQ1 container, reference divuq.io)
from .parallel import BenchReport, bench, parallel_map
from .api import (
    EnsembleDivergence,
    cell_crossing_probability,
    gradient,
    gradient_ensemble,
    gradient_ensemble_divergence,
    lcp,
    velocity_magnitude,
    Propagation,
    divergence_deterministic,
    ensemble_divergence,
    ensemble_divergence3d,
    error_metrics,
    fit_gaussian,
    mc_divergence,
    mc_histogram_1d,
    propagate_divergence,
    propagate_lcp,
    propagate_with_probabilities,
    propagate_with_probabilities3d,
    set_device,
    sink_probability,
    source_probability,
    sample_divergence_1d,
    stencil_distribution,
    tail_probs,
)
from .types import (
    Ensemble2,
    GaussianScalarField,
    GaussianScalarField3,
    GaussianVectorField,
    GaussianVectorField3,
    LcpField,
    McConfig,
    McDivergenceEstimate,
    McHistogram,
    ParallelConfig,
    ScalarField2,
    UniformGrid2,
    UniformGrid3,
    VectorField2,
    vertex_index,
)

__version__ = "0.1.0"

__all__ = [
    "BenchReport", "bench", "parallel_map", "Ensemble2", "EnsembleDivergence",
    "GaussianScalarField", "GaussianScalarField3", "GaussianVectorField",
    "GaussianVectorField3", "LcpField", "McConfig", "McDivergenceEstimate", "McHistogram",
    "ParallelConfig", "Propagation", "ScalarField2", "UniformGrid2", "UniformGrid3",
    "VectorField2", "cell_crossing_probability", "divergence_deterministic",
    "ensemble_divergence", "ensemble_divergence3d", "gradient_ensemble_divergence",
    "error_metrics", "fit_gaussian", "gradient", "gradient_ensemble", "lcp", "propagate_lcp",
    "mc_divergence",
    "mc_histogram_1d", "sample_divergence_1d", "velocity_magnitude", "propagate_divergence",
    "propagate_with_probabilities", "propagate_with_probabilities3d", "set_device",
    "sink_probability", "source_probability", "stencil_distribution", "tail_probs",
    "vertex_index",
]
