"""B200-native DELIMIT spherical-signal layers (arXiv 1808.01517).

Signal2SH, SH2Signal and LocalSphericalConvolution as torch.nn.Modules over
hand-written sm_100a CUDA kernels (libdelimit_sm100a.so, C ABI in
include/delimit.h), plus a fused SphericalChain and a drop-in functional API
mirroring the reference implementation (sphdwi 0.1.0).
"""

from .errors import (
    DelimitError,
    DeviceError,
    GradientParseError,
    IllPosedFitError,
    KernelMismatchError,
    MissingB0Error,
    NiftiDatatypeError,
    NiftiError,
    NiftiMagicError,
    NiftiTruncatedError,
    ShapeError,
    SphdwiError,
)
from .geometry import (
    SH_C0,
    TWO_SQRT_PI,
    FitOperator,
    LscGeometry,
    LscKernel,
    ShBasisSpec,
    as_unit_directions,
    basis_degrees,
    build_lsc_geometry,
    coeff_count,
    degree_energies,
    eval_basis,
    high_degree_energy_fraction,
    laplace_beltrami_diag,
    make_fit_operator,
    make_identity_kernel,
    make_moving_average_kernel,
    ring_directions,
    sh_degree_order,
    sh_index,
    tangent_basis,
)
from .modules import LocalSphericalConvolution, RoundTrip, SH2Signal, Signal2SH, SphericalChain, SphericalKernel
from .functional import (
    DwiVolume,
    ShVolume,
    apply_channel_matrix,
    lsc_combine,
    lsc_forward,
    sh_to_signal,
    signal_to_sh,
)

from . import dwio
from .ingest import chain_from_raw, load_dwi, normalize_b0

__version__ = "0.1.0"


def library_path() -> str:
    from ._lib import LIB_PATH

    return LIB_PATH
