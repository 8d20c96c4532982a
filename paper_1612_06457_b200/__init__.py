"""B200-native CVA / PCA hot path of arXiv:1612.06457 ("undertext").

Drop-in for the hot-path functions of the reference package ``undertext``
(/root/reference/pkg/src/undertext): same names, signatures, return types and
errors, computed by hand-written sm_100a kernels behind the C ABI in
``include/undertext_b200.h`` (library: ``paper_1612_06457_b200/lib``).
There is no CPU fallback: compute entry points raise if the library or a CUDA
device is missing.
"""

from .annotations import (AnnotatedPoint, ClassLabel, DesignMatrix, TrainingSet,  # noqa: F401
                          assemble_matrix)
from .eigen import (DEFAULT_RIDGE, EigenSolution, regularize, sign_normalize,  # noqa: F401
                    solve_gen_eig_sym)
from .image_io import encode_png, encode_tiff, load_image, save_image  # noqa: F401
from .errors import DataError, NumericError, UndertextError, UndertextWarning  # noqa: F401
from .pipeline import (CvaPipeline, FolioStream, PcaPipeline, RenderResult,  # noqa: F401
                       composite_filename, fit_model, load_normalized, model_provenance,
                       plane_filename, project_single, render_planes, route_points,
                       row_bounds)
from .projection import (ALL_METHODS, METHOD_CVA, METHOD_LDA, METHOD_PCA,  # noqa: F401
                         METHOD_PCA_UNSUPERVISED, ProjectionModel, ScatterPair,
                         compute_scatter, fit, fit_cva, fit_lda, fit_pca,
                         fit_pca_unsupervised, project_stack, standardize)
from .quantize import code_dtype, linear_to_codes, max_code, round_half_away  # noqa: F401
from .rendering import (PERCENTILE_CHOICES, CompositeRecipe, DeviceScorePlane,  # noqa: F401
                        RenderSpec, compose_rgb,
                        ScorePlane, nearest_rank_percentile, rescale, rescale_full,
                        rescale_percentile, rescale_training_range)
from .stack import (BandMeta, DeviceStack, SpectralStack, crop, load_device_stack,  # noqa: F401
                    load_stack, normalize_stack)

__version__ = "0.1.0"
