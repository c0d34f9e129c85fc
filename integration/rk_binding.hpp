// Helpers shared by the reference-side binding files (projector_b200.cpp,
// sino_filter_b200.cpp): radonkit::Tensor <-> C-ABI buffers, status -> the
// reference's exception types (errors.hpp), and the per-geometry plan cache.
#pragma once

#include "radon_b200.h"
#include "radonkit/geometry.hpp"
#include "radonkit/tensor.hpp"

namespace radonkit::b200 {

int dtype_of(const Tensor& t);        // Precision -> RK_F16 / RK_F32 / RK_F64
const void* data_of(const Tensor& t);  // the storage vector's buffer
void* data_of(Tensor& t);
void check(int status);  // RK_ERR_VALIDATION -> ValidationError, RK_ERR_NUMERICAL -> NumericalError
int device();            // $RK_DEVICE, default 0

// Process-wide plan per (geometry, step); plans live until exit.
rk_plan* plan_for(const ParallelGeometry& g, double step);
rk_plan* plan_for(const FanbeamGeometry& g, double step);

}  // namespace radonkit::b200
