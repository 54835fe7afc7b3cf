// k1d.cuh -- 1-D (and batched) running max-min filter kernels for sm_100a.
// The kernels live in k1d_small.cuh, k1d_medium.cuh and k1d_large.cuh; the
// shared design notes and helpers are in k1d_base.cuh.
#pragma once

#include "k1d_base.cuh"
#include "k1d_small.cuh"
#include "k1d_medium.cuh"
#include "k1d_large.cuh"
#include "k1d_warp.cuh"
#include "k1d_lw.cuh"
