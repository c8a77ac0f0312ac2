// finalize + texel_argmax (fusion.py:186-222), render_labels
// (renderback.py:28-56) and the per-pixel network argmax (cli.py:293).
#include <math.h>

#include "common.cuh"

namespace tfb {
namespace {

// NumPy argmax order: the first NaN wins, otherwise the first maximum.
__device__ __forceinline__ bool better(float a, int ia, float b, int ib) {
  const bool na = isnan(a), nb = isnan(b);
  if (na || nb) return na && (!nb || ia < ib);
  return a > b || (a == b && ia < ib);
}

template <typename AccT>
__global__ void __launch_bounds__(256) k_finalize(const AccT *__restrict__ accum, int64_t stride,
                                                  const uint32_t *__restrict__ counts, int64_t n_x, int c, int agg,
                                                  float *rows_out, uint8_t *unobs_out, int32_t *labels_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_x; i += nwarps) {
    const AccT *a = accum + i * stride;
    const bool zero_count = counts[i] == 0u;
    bool unobs;
    double scale, shift = 0.0;
    if (agg == TFB_AGG_MUL) {
      // rows = exp(accum - rowmax) / sum  (fusion.py:196-200)
      double mx = -INFINITY;
      for (int k = lane; k < c; k += 32) mx = fmax(mx, (double)a[k]);
#pragma unroll
      for (int d = 16; d; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      double s = 0.0;
      for (int k = lane; k < c; k += 32) s += exp((double)a[k] - mx);
#pragma unroll
      for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
      shift = mx;
      scale = s;
      unobs = zero_count;
    } else {
      // rows = accum / L1 norm; zero mass counts as unobserved (fusion.py:202-205)
      double s = 0.0;
      for (int k = lane; k < c; k += 32) s += (double)a[k];
#pragma unroll
      for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
      unobs = zero_count || !(s > 0.0);
      scale = s > 0.0 ? s : 1.0;
    }
    const float uni = (float)(1.0 / c);
    float bv = 0.f;
    int bi = 0x7fffffff;
    for (int k = lane; k < c; k += 32) {
      float v;
      if (unobs) v = uni;
      else if (agg == TFB_AGG_MUL) v = (float)(exp((double)a[k] - shift) / scale);
      else v = (float)((double)a[k] / scale);
      if (rows_out) rows_out[i * c + k] = v;
      if (bi == 0x7fffffff || better(v, k, bv, bi)) {
        bv = v;
        bi = k;
      }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, d);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
      if (oi != 0x7fffffff && (bi == 0x7fffffff || better(ov, oi, bv, bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      if (unobs_out) unobs_out[i] = unobs ? 1 : 0;
      if (labels_out) labels_out[i] = unobs ? -1 : bi;
    }
  }
}

__global__ void k_render(const int32_t *rows, int64_t n, const int32_t *labels, const int32_t *fallback, int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[i];
    int32_t v = r >= 0 ? __ldg(labels + r) : -1;
    if (fallback && v == -1) v = fallback[i];
    out[i] = v;
  }
}

__global__ void k_probs_argmax(const float *probs, int64_t npix, int c, int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
    const float *pp = probs + i * c;
    float best = pp[0];
    int bi = 0;
    for (int k = 1; k < c; ++k) {
      const float v = pp[k];
      if (!isnan(best) && (isnan(v) || v > best)) {
        best = v;
        bi = k;
      }
    }
    out[i] = bi;
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 8192) b = 8192;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace
}  // namespace tfb

using namespace tfb;

extern "C" int tfb_finalize(const void *accum, int accum_is_f64, int64_t accum_stride, const uint32_t *counts,
                            int64_t total_texels, int num_classes, int aggregator, float *rows_out,
                            uint8_t *unobserved_out, int32_t *labels_out, void *stream) {
  TFB_REQUIRE(aggregator >= 0 && aggregator <= 2, TFB_ERR_VALUE, "unknown aggregator id %d", aggregator);
  TFB_REQUIRE(num_classes >= 1 && accum_stride >= num_classes, TFB_ERR_DATA, "tfb_finalize: bad class count/stride");
  TFB_REQUIRE(accum && counts, TFB_ERR_DATA, "tfb_finalize: null accum or counts");
  if (total_texels <= 0) return TFB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = (total_texels + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (accum_is_f64)
    k_finalize<double><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const double *>(accum), accum_stride, counts,
                                                          total_texels, num_classes, aggregator, rows_out,
                                                          unobserved_out, labels_out);
  else
    k_finalize<float><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const float *>(accum), accum_stride, counts,
                                                         total_texels, num_classes, aggregator, rows_out,
                                                         unobserved_out, labels_out);
  return check_launch("tfb_finalize");
}

extern "C" int tfb_render(const int32_t *rows, int64_t hw, int nframes, const int32_t *texel_labels,
                          int64_t total_texels, const int32_t *fallback, int32_t *out, void *stream) {
  (void)total_texels;
  TFB_REQUIRE(rows && texel_labels && out, TFB_ERR_DATA, "tfb_render: null argument");
  const int64_t n = hw * (int64_t)nframes;
  if (n <= 0) return TFB_OK;
  k_render<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, n, texel_labels, fallback, out);
  return check_launch("tfb_render");
}

extern "C" int tfb_probs_argmax(const float *probs, int64_t npix, int num_classes, int32_t *out, void *stream) {
  TFB_REQUIRE(probs && out && num_classes >= 1, TFB_ERR_DATA, "tfb_probs_argmax: bad argument");
  if (npix <= 0) return TFB_OK;
  k_probs_argmax<<<grid_for(npix), 256, 0, static_cast<cudaStream_t>(stream)>>>(probs, npix, num_classes, out);
  return check_launch("tfb_probs_argmax");
}
