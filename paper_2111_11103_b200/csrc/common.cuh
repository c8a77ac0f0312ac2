// Shared helpers for the sm_100a kernels of texelfuse_b200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "texelfuse_b200.h"

namespace tfb {

constexpr double kNearPlane = 1e-4;  // geometry.py:26
constexpr double kDepthTie = 1e-9;   // rasterizer.py:18
constexpr float kMulClampF = 1e-7f;  // fusion.py:39
constexpr double kMulClamp = 1e-7;   // fusion.py:39

void set_error(const char *fmt, ...);

// Returns TFB_ERR_CUDA (with message) if the last launch failed.
int check_launch(const char *what);

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace tfb

#define TFB_REQUIRE(cond, code, ...)     \
  do {                                   \
    if (!(cond)) {                       \
      ::tfb::set_error(__VA_ARGS__);     \
      return code;                       \
    }                                    \
  } while (0)
