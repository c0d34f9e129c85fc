"""B200-native (sm_100a) drop-in for TorchRadon's hot path: batched
parallel-beam and fan-beam Radon forward projection, its adjoint
backprojection and ramp-filtered backprojection.

The Python surface mirrors the reference's operator API ("radonkit",
``/root/reference/proj/core/include/radonkit``): geometry makers,
``forward`` / ``backprojection``, ``make_filter`` / ``filter_sinogram`` /
``fbp``, the ``LinearOperator`` wrapper and the iterative solvers.  Every
call goes through the C ABI (``include/radon_b200.h``) of the in-tree CUDA
library ``libradon_b200.so``; there is no CPU fallback.
"""
from .errors import (CudaError, DivergenceError, HalfOverflowError, NotPositiveDefiniteError, NumericalError,
                     ValidationError)
from .geometry import (FanbeamGeometry, Geometry, ParallelGeometry, angles_linspace, geometry_det_count,
                       geometry_image_size, geometry_n_angles, make_fanbeam, make_parallel)
from .projector import ProjectorOptions, backprojection, get_plan, materialize_matrix
from .projector import forward as _projector_forward
from .sino_filter import FilterKind, FilterSpec, fbp, filter_kind_from_name, filter_kind_name, filter_sinogram, make_filter
from .linop import (LinearOperator, adjoint_check, compose, gradient_check, identity_operator, projector_operator)
from .rng import Rng
from .solvers import cg, cgne, estimate_alpha, landweber
from . import shearlet
from .shearlet import ShearletPlan, backward, make_plan, make_plan_cached, shearlet_operator
from .admm import AdmmParams, AdmmState, admm_objective, admm_reconstruct, default_weights, shrink
from .npy import read_array, write_array
from .png_io import png_export
from .threading import num_threads, set_num_threads


def forward(plan_or_geometry, x, *args, **kwargs):
    """The reference's two ``forward`` overloads: Radon projection
    (projector.hpp, ``forward(geometry, image[, opts])``) and shearlet analysis
    (shearlet.hpp:49, ``forward(plan, image)``)."""
    if isinstance(plan_or_geometry, ShearletPlan):
        return shearlet.forward(plan_or_geometry, x, *args, **kwargs)
    return _projector_forward(plan_or_geometry, x, *args, **kwargs)


__all__ = [
    "CudaError", "DivergenceError", "HalfOverflowError", "NotPositiveDefiniteError", "NumericalError",
    "ValidationError", "FanbeamGeometry", "Geometry", "ParallelGeometry", "angles_linspace", "geometry_det_count",
    "geometry_image_size", "geometry_n_angles", "make_fanbeam", "make_parallel", "ProjectorOptions",
    "backprojection", "forward", "get_plan", "materialize_matrix", "FilterKind", "FilterSpec", "fbp", "filter_kind_from_name",
    "filter_kind_name", "filter_sinogram", "make_filter", "LinearOperator", "adjoint_check", "compose",
    "gradient_check", "identity_operator", "projector_operator", "Rng", "cg", "cgne", "estimate_alpha", "landweber",
    "ShearletPlan", "backward", "make_plan", "make_plan_cached", "shearlet", "shearlet_operator",
    "AdmmParams", "AdmmState", "admm_objective", "admm_reconstruct", "default_weights", "shrink",
    "read_array", "write_array", "png_export", "num_threads", "set_num_threads",
]
