"""B200-native (sm_100a) log-polar fast backprojection — drop-in for the fastbp
backprojection / FBP path of arXiv 1608.03589 (reference package pkg/src/fastbp).

Same names and signatures as the reference for the path:
  Sinogram, CartesianImage, LogPolarImage, LogPolarOptions, FilterSpec,
  logpolar_backproject, filter_sinogram, fbp, backproject_naive,
  adaptive_rho0, compute_nrho, relative_l2, partial_backproject,
  BstOptions, bst_backproject (fbp's default engine "bst"),
  PolarSinogram, sinogram_to_semipolar, semipolar_to_logpolar, logpolar_to_cartesian,
  make_logpolar_kernel, truncation_error_bound,
  Ellipse, EllipseSet, radon_ellipses (the input generator, on the device)
plus batched device entry points (torch CUDA tensors) and LogPolarPlan.
All compute runs in liblpbp.so; there is no CPU fallback.
"""

from .grids import CartesianImage, LogPolarImage, Sinogram, adaptive_rho0, compute_nrho
from .logpolar import (
    LOGPOLAR_SCALE,
    LogPolarOptions,
    logpolar_backproject,
    logpolar_backproject_batch,
    logpolar_convolve,
    mesh_for,
)
from .filtering import FBP_SCALE, FilterSpec, fbp, fbp_batch, filter_sinogram
from .reference import backproject_naive, backproject_naive_batch
from .metrics import max_abs_error, relative_l2
from .plan import LogPolarPlan, get_plan, naive_backproject
from .roofline import algorithmic_bytes
from . import roofline
from . import synth
from .synth import Ellipse, EllipseSet, radon_ellipses
from .multi import VolumeReconstructor, shard_bounds
from .sector import SectorPlan, partial_backproject, partial_backproject_batch
from .bst import (
    BST_SCALE,
    BstOptions,
    BstPlan,
    bst_backproject,
    bst_backproject_batch,
    bst_spectrum,
    kaiser_window,
    mean_backprojection,
    sigma_kernel,
)
from .resample import (
    FrequencyImage,
    PolarSinogram,
    PolarSpectrum,
    polar_to_cartesian_frequency,
    logpolar_to_cartesian,
    make_logpolar_kernel,
    semipolar_to_logpolar,
    sinogram_to_semipolar,
    truncation_error_bound,
)

__version__ = "0.1.0"
