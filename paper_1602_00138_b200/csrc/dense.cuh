// Dense tall-skinny block kernels (Gram, block GEMM, small on-device
// factorisations) -- filled in with the CholQR2 refresh and RRQR.
#pragma once
#include "common.cuh"
