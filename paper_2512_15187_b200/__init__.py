"""B200-native (sm_100a) Probabilistic Inclusion Depth — drop-in for the depth
hot path of the reference package ``fuzzdepth`` (arXiv 2512.15187).

Same entry points as the reference (depth_pid, depth_pid_mean, depth_eid,
depth_by_method, prob_inclusion, subset_epsilon, member_masses, mean_mask,
mask_mass, DepthResult, ranks_from_depths, and the GridSpec / ProbMask /
BinaryMask / Ensemble containers); the arithmetic runs in hand-written CUDA
kernels in ``libpidb.so`` (C ABI: include/pidb.h).  No CPU fallback.
"""
from .depth import (
    CV_WARN_THRESHOLD,
    METHOD_NAMES,
    DepthResult,
    compare_pid_vs_mean,
    depth_by_method,
    depth_eid,
    depth_pid,
    depth_pid_mean,
    depth_similarity_baseline,
    mass_cv,
    member_masses,
    ranks_from_depths,
    resolve_workers,
)
from .device import DeviceEnsemble, shard_bounds, stage
from .errors import (
    DegenerateEnsembleError,
    FuzzdepthError,
    GridMismatchError,
    ManifestError,
    ValidationError,
    VolumeFormatError,
)
from .grid import (
    BinaryMask,
    Ensemble,
    GridSpec,
    ProbMask,
    binarize,
    binarize_ensemble,
    binary_mass,
    mask_mass,
    mean_mask,
    permute_cells,
)
from .inclusion import fuzzy_dice, prob_inclusion, prob_iou, subset_epsilon
from .reduction import gram_block
from .synth import (gen_contour_ensemble_2d, gen_disk_ensemble, gen_ellipsoid_ensemble,
                    gen_fuzzy_disk)
from .io import ScalarField
from .boxplot import Band, BoxplotArtifact, build_boxplot, emit_slice_images, write_pgm
from .consistency import RankScatter, kendall_tau, pearson, rank_scatter, stability_test
from .io import (manifest_guarantees_binary, read_depth_csv, read_manifest, read_volume,
                 stage_manifest, volume_header, write_boxplot_artifact, write_depth_csv,
                 write_manifest, write_scatter_csv, write_volume)

__version__ = "0.1.0"

__all__ = [
    "Band",
    "BoxplotArtifact",
    "RankScatter",
    "ScalarField",
    "build_boxplot",
    "emit_slice_images",
    "kendall_tau",
    "manifest_guarantees_binary",
    "pearson",
    "rank_scatter",
    "read_depth_csv",
    "read_manifest",
    "read_volume",
    "stability_test",
    "stage_manifest",
    "volume_header",
    "write_boxplot_artifact",
    "write_depth_csv",
    "write_manifest",
    "write_pgm",
    "write_scatter_csv",
    "write_volume",
    "BinaryMask",
    "CV_WARN_THRESHOLD",
    "DegenerateEnsembleError",
    "DepthResult",
    "DeviceEnsemble",
    "Ensemble",
    "FuzzdepthError",
    "GridMismatchError",
    "GridSpec",
    "ManifestError",
    "METHOD_NAMES",
    "ProbMask",
    "ValidationError",
    "VolumeFormatError",
    "binarize",
    "binarize_ensemble",
    "binary_mass",
    "compare_pid_vs_mean",
    "depth_by_method",
    "depth_eid",
    "depth_pid",
    "depth_pid_mean",
    "depth_similarity_baseline",
    "fuzzy_dice",
    "gen_contour_ensemble_2d",
    "gen_disk_ensemble",
    "gen_ellipsoid_ensemble",
    "gen_fuzzy_disk",
    "gram_block",
    "mask_mass",
    "mass_cv",
    "mean_mask",
    "member_masses",
    "permute_cells",
    "prob_inclusion",
    "prob_iou",
    "ranks_from_depths",
    "resolve_workers",
    "shard_bounds",
    "stage",
    "subset_epsilon",
    "__version__",
]
