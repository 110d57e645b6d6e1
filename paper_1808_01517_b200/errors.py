"""Exception types, mirroring the reference's taxonomy (sphdwi/errors.py:8-45).

The same conditions raise the same classes as the reference: channel / order /
shell mismatches -> ShapeError, kernel length mismatch -> KernelMismatchError,
ill-posed fits -> IllPosedFitError, bad scalar arguments -> ValueError.
DeviceError is new: the path is CUDA-only and fails loudly without it.
"""


class SphdwiError(Exception):
    """Base class for all package-specific errors (reference name kept for drop-in use)."""


DelimitError = SphdwiError


class ShapeError(SphdwiError):
    """An array does not have the channel/volume layout an operation expects."""


class IllPosedFitError(SphdwiError):
    """The least-squares system is underdetermined or numerically rank deficient."""


class KernelMismatchError(SphdwiError):
    """A convolution kernel does not match the geometry it is applied with."""


class DeviceError(SphdwiError, RuntimeError):
    """No sm_100a device, missing CUDA library, or a CUDA error from the kernels."""


class MissingB0Error(SphdwiError):
    """The acquisition has no b=0 volume to normalise against (errors.py:20-21)."""


class GradientParseError(SphdwiError):
    """A bvals / bvecs table is malformed or inconsistent (errors.py:24-25)."""


class NiftiError(SphdwiError):
    """Base class for NIfTI-1 read/write failures (errors.py:32-33)."""


class NiftiMagicError(NiftiError):
    """Not a single-file NIfTI-1 (bad sizeof_hdr / magic / dimensions / vox_offset)."""


class NiftiDatatypeError(NiftiError):
    """Unsupported voxel datatype code."""


class NiftiTruncatedError(NiftiError):
    """The file ends before the header or the voxel data it promises."""
