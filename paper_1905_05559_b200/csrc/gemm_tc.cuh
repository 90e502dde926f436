// gemm_tc.cuh -- tcgen05 (TF32) GEMM for the curvature products.
#pragma once
#include "curvature.cuh"
