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

// One group of L lanes per texel (L = 8 when c <= 64, so four texels per warp
// are in flight; L = 32 above).  The exponentials of the product rule are kept
// in registers between the sum and the rows (up to kKeep per lane).
constexpr int kKeep = 8;

// accumulator element as float64 (TFB_ACCUM_FIXED elements are value * 2^32)
__device__ __forceinline__ double acc_val(float x) { return (double)x; }
__device__ __forceinline__ double acc_val(double x) { return x; }
__device__ __forceinline__ double acc_val(long long x) { return (double)x * 2.3283064365386963e-10; }

template <typename AccT, int L>
__global__ void __launch_bounds__(256) k_finalize(const AccT *__restrict__ accum, int64_t stride,
                                                  const uint32_t *__restrict__ counts, int64_t n_x, int c, int agg,
                                                  float *rows_out, uint8_t *unobs_out, int32_t *labels_out) {
  const int sub = threadIdx.x & (L - 1);
  const int64_t ngroups = (int64_t)gridDim.x * (blockDim.x / L);
  const int64_t first = (int64_t)blockIdx.x * (blockDim.x / L) + (threadIdx.x / L);
  // every lane runs the same number of iterations (shuffles stay converged)
  const int64_t iters = (n_x + ngroups - 1) / ngroups;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = first + it * ngroups;
    const bool live = i < n_x;
    const AccT *a = accum + (live ? i : 0) * stride;
    const bool zero_count = live ? counts[i] == 0u : true;
    bool unobs;
    double scale, shift = 0.0;
    double ex[kKeep];
    if (agg == TFB_AGG_MUL) {
      // rows = exp(accum - rowmax) / sum  (fusion.py:196-200)
      double mx = -INFINITY;
      for (int k = sub; k < c; k += L) mx = fmax(mx, acc_val(a[k]));
#pragma unroll
      for (int d = L / 2; d; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d, L));
      double sacc = 0.0;
#pragma unroll
      for (int kk = 0; kk < kKeep; ++kk) {
        const int k = sub + kk * L;
        ex[kk] = k < c ? exp(acc_val(a[k]) - mx) : 0.0;
        sacc += ex[kk];
      }
      for (int k = sub + kKeep * L; k < c; k += L) sacc += exp(acc_val(a[k]) - mx);
#pragma unroll
      for (int d = L / 2; d; d >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, d, L);
      shift = mx;
      scale = sacc;
      unobs = zero_count;
    } else {
      // rows = accum / L1 norm; zero mass counts as unobserved (fusion.py:202-205)
      double sacc = 0.0;
      for (int k = sub; k < c; k += L) sacc += acc_val(a[k]);
#pragma unroll
      for (int d = L / 2; d; d >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, d, L);
      unobs = zero_count || sacc <= 0.0;  // a NaN mass stays observed, rows = accum / 1 (fusion.py:203-205)
      scale = sacc > 0.0 ? sacc : 1.0;
    }
    const float uni = (float)(1.0 / c);
    float bv = 0.f;
    int bi = 0x7fffffff;
    for (int k = sub, kk = 0; k < c; k += L, ++kk) {
      float v;
      if (unobs) {
        v = uni;
      } else if (agg == TFB_AGG_MUL) {
        double e;
        if (kk < kKeep) {
          e = 0.0;
#pragma unroll
          for (int q = 0; q < kKeep; ++q) e = q == kk ? ex[q] : e;
        } else {
          e = exp(acc_val(a[k]) - shift);
        }
        v = (float)(e / scale);
      } else {
        v = (float)(acc_val(a[k]) / scale);
      }
      if (rows_out && live) rows_out[i * c + k] = v;
      if (bi == 0x7fffffff || better(v, k, bv, bi)) {
        bv = v;
        bi = k;
      }
    }
#pragma unroll
    for (int d = L / 2; d; d >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, d, L);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, d, L);
      if (oi != 0x7fffffff && (bi == 0x7fffffff || better(ov, oi, bv, bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if (sub == 0 && live) {
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

extern "C" int tfb_finalize(const void *accum, int accum_kind, int64_t accum_stride, const uint32_t *counts,
                            int64_t total_texels, int num_classes, int aggregator, float *rows_out,
                            uint8_t *unobserved_out, int32_t *labels_out, void *stream) {
  TFB_REQUIRE(aggregator >= 0 && aggregator <= 2, TFB_ERR_VALUE, "unknown aggregator id %d", aggregator);
  TFB_REQUIRE(num_classes >= 1 && accum_stride >= num_classes, TFB_ERR_DATA, "tfb_finalize: bad class count/stride");
  TFB_REQUIRE(accum && counts, TFB_ERR_DATA, "tfb_finalize: null accum or counts");
  if (total_texels <= 0) return TFB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool narrow = num_classes <= 64;  // 8 lanes per texel
  const int64_t per_block = narrow ? 32 : 8;
  int64_t blocks = (total_texels + per_block - 1) / per_block;
  if (blocks > 148 * 64) blocks = 148 * 64;
  const unsigned g = (unsigned)blocks;
  TFB_REQUIRE(accum_kind >= TFB_ACCUM_F32 && accum_kind <= TFB_ACCUM_FIXED, TFB_ERR_VALUE,
              "unknown accumulator kind %d", accum_kind);
  if (accum_kind == TFB_ACCUM_FIXED) {
    const long long *a = static_cast<const long long *>(accum);
    if (narrow)
      k_finalize<long long, 8><<<g, 256, 0, st>>>(a, accum_stride, counts, total_texels, num_classes, aggregator,
                                                  rows_out, unobserved_out, labels_out);
    else
      k_finalize<long long, 32><<<g, 256, 0, st>>>(a, accum_stride, counts, total_texels, num_classes, aggregator,
                                                   rows_out, unobserved_out, labels_out);
  } else if (accum_kind == TFB_ACCUM_F64) {
    const double *a = static_cast<const double *>(accum);
    if (narrow)
      k_finalize<double, 8><<<g, 256, 0, st>>>(a, accum_stride, counts, total_texels, num_classes, aggregator,
                                               rows_out, unobserved_out, labels_out);
    else
      k_finalize<double, 32><<<g, 256, 0, st>>>(a, accum_stride, counts, total_texels, num_classes, aggregator,
                                                rows_out, unobserved_out, labels_out);
  } else {
    const float *a = static_cast<const float *>(accum);
    if (narrow)
      k_finalize<float, 8><<<g, 256, 0, st>>>(a, accum_stride, counts, total_texels, num_classes, aggregator,
                                              rows_out, unobserved_out, labels_out);
    else
      k_finalize<float, 32><<<g, 256, 0, st>>>(a, accum_stride, counts, total_texels, num_classes, aggregator,
                                               rows_out, unobserved_out, labels_out);
  }
  return check_launch("tfb_finalize");
}

extern "C" int tfb_render(const int32_t *rows, int64_t hw, int nframes, const int32_t *texel_labels,
                          int64_t total_texels, const int32_t *fallback, int32_t *out, void *stream) {
  // an empty layout has no labels (every row is -1): texel_labels may then be NULL
  TFB_REQUIRE(rows && out && (texel_labels || total_texels == 0), TFB_ERR_DATA, "tfb_render: null argument");
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
