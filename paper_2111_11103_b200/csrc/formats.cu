// Device kernels for the data formats and reports either side of the hot path
// (SURVEY §8(f) #2-#4):
//   k_probs_check   SMPB load validation (formats.py:77-93): global minimum and
//                   the largest |sum_k p - 1| over pixels, sums in float64.
//   k_confusion     pixel_accuracy (renderback.py:152-172): confusion matrix,
//                   per-class unknown predictions, ignored reference pixels.
//   k_face_majority export_colored_mesh (renderback.py:275-294): per-face vote
//                   over the labels of its texels, first maximum wins.
#include <math.h>

#include "common.cuh"

namespace tfb {
namespace {

// order-preserving 64-bit key of a double (for atomicMin over signed values)
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double from_order_key(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// NumPy's float64 add-reduce of one contiguous row: out = a[0], then the
// remaining n-1 values by pairwise summation (8 interleaved partial sums in
// blocks of up to 128, halves above that), as numpy/_core/src/umath/loops_utils.h.
__device__ double np_pairwise(const float *a, int n) {
  if (n < 8) {
    double r = 0.0;  // n < 8: plain left-to-right sum (only -0.0 differs from the identity)
    for (int i = 0; i < n; ++i) r += (double)a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (double)a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += (double)a[i + j];
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += (double)a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

// state[0]: min order key, state[1]: max |err| bits, state[2]: NaN in values, state[3]: NaN in sums
__global__ void k_probs_check_init(unsigned long long *state) {
  state[0] = ~0ull;
  state[1] = 0ull;
  state[2] = 0ull;
  state[3] = 0ull;
}

__global__ void __launch_bounds__(256) k_probs_check(const float *__restrict__ probs, int64_t npix, int c,
                                                     unsigned long long *state) {
  unsigned long long kmin = ~0ull, emax = 0ull;
  bool nan_v = false, nan_e = false;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    const float *row = probs + p * c;
    float mn = row[0];
    for (int k = 1; k < c; ++k) mn = fminf(mn, row[k]);
    for (int k = 0; k < c; ++k) nan_v |= isnan(row[k]);
    const double s = c > 1 ? (double)row[0] + np_pairwise(row + 1, c - 1) : (double)row[0];
    const double e = fabs(s - 1.0);
    nan_e |= isnan(e);
    const unsigned long long km = order_key((double)mn);
    kmin = km < kmin ? km : kmin;
    const unsigned long long eb = (unsigned long long)__double_as_longlong(e);
    if (!isnan(e) && eb > emax) emax = eb;
  }
  // warp then one atomic per warp
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long ok = __shfl_down_sync(0xffffffffu, kmin, d);
    const unsigned long long oe = __shfl_down_sync(0xffffffffu, emax, d);
    kmin = ok < kmin ? ok : kmin;
    emax = oe > emax ? oe : emax;
  }
  nan_v = __any_sync(0xffffffffu, nan_v);
  nan_e = __any_sync(0xffffffffu, nan_e);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(state, kmin);
    atomicMax(state + 1, emax);
    if (nan_v) atomicOr(state + 2, 1ull);
    if (nan_e) atomicOr(state + 3, 1ull);
  }
}

__global__ void k_probs_check_fin(unsigned long long *state) {
  double *out = reinterpret_cast<double *>(state);
  const double mn = state[2] ? __longlong_as_double(0x7ff8000000000000LL) : from_order_key(state[0]);
  const double er = state[3] ? __longlong_as_double(0x7ff8000000000000LL) : __longlong_as_double((long long)state[1]);
  out[0] = mn;
  out[1] = er;
}

constexpr int kConfSmem = 4096;  // c*c bins kept in shared memory up to c = 64

__global__ void __launch_bounds__(256) k_confusion(const int32_t *__restrict__ pred, const int32_t *__restrict__ ref,
                                                   int64_t npix, int c, const uint8_t *__restrict__ ignore,
                                                   unsigned long long *confusion, unsigned long long *unknown,
                                                   unsigned long long *valid_count) {
  __shared__ unsigned int hist[kConfSmem];
  __shared__ unsigned int unk[256];
  __shared__ unsigned int nvalid;
  const bool local = c * c <= kConfSmem && c <= 256;
  if (local) {
    for (int i = threadIdx.x; i < c * c; i += blockDim.x) hist[i] = 0u;
    for (int i = threadIdx.x; i < c; i += blockDim.x) unk[i] = 0u;
  }
  if (threadIdx.x == 0) nvalid = 0u;
  __syncthreads();
  unsigned int my_valid = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = ref[i];
    if (g < 0 || g >= c || (ignore && ignore[g])) continue;  // renderback.py:160-163
    ++my_valid;
    const int p = pred[i];
    const bool known = p >= 0 && p < c;
    if (local) {
      if (known) atomicAdd(hist + g * c + p, 1u);
      else atomicAdd(unk + g, 1u);
    } else {
      if (known) atomicAdd(confusion + (int64_t)g * c + p, 1ull);
      else atomicAdd(unknown + g, 1ull);
    }
  }
  atomicAdd(&nvalid, my_valid);
  __syncthreads();
  if (local) {
    for (int i = threadIdx.x; i < c * c; i += blockDim.x)
      if (hist[i]) atomicAdd(confusion + i, (unsigned long long)hist[i]);
    for (int i = threadIdx.x; i < c; i += blockDim.x)
      if (unk[i]) atomicAdd(unknown + i, (unsigned long long)unk[i]);
  }
  if (threadIdx.x == 0 && nvalid) atomicAdd(valid_count, (unsigned long long)nvalid);
}

// warp per face; votes of the face's texels in a per-warp shared-memory histogram
__global__ void __launch_bounds__(256) k_face_majority(const int32_t *__restrict__ labels,
                                                       const int32_t *__restrict__ steps,
                                                       const int64_t *__restrict__ offsets, int64_t m, int c,
                                                       int32_t *face_class) {
  extern __shared__ unsigned int fhist[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int *h = fhist + (size_t)warp * c;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; t < m; t += wstride) {
    for (int k = lane; k < c; k += 32) h[k] = 0u;
    __syncwarp();
    const int64_t s = steps[t];
    const int64_t cnt = (s * s + s) / 2;
    const int64_t o = offsets[t];
    unsigned int nv = 0;
    for (int64_t i = lane; i < cnt; i += 32) {
      const int l = labels[o + i];
      if (l >= 0 && l < c) {
        atomicAdd(h + l, 1u);
        ++nv;
      }
    }
    for (int d = 16; d > 0; d >>= 1) nv += __shfl_down_sync(0xffffffffu, nv, d);
    __syncwarp();
    // argmax with the first maximum winning (np.argmax over the vote row)
    unsigned int best = 0u;
    int bi = 0x7fffffff;
    for (int k = lane; k < c; k += 32) {
      const unsigned int v = h[k];
      if (v > best || (v == best && k < bi)) {
        best = v;
        bi = k;
      }
    }
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned int ov = __shfl_down_sync(0xffffffffu, best, d);
      const int oi = __shfl_down_sync(0xffffffffu, bi, d);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) face_class[t] = nv ? bi : -1;  // -1: no observed texel (UNOBSERVED_GRAY)
    __syncwarp();
  }
}

}  // namespace
}  // namespace tfb

using namespace tfb;

extern "C" int tfb_probs_check(const float *probs, int64_t npix, int num_classes, double *out4, void *stream) {
  TFB_REQUIRE(probs && out4, TFB_ERR_DATA, "tfb_probs_check: null argument");
  TFB_REQUIRE(num_classes >= 1, TFB_ERR_VALUE, "num_classes must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long *state = reinterpret_cast<unsigned long long *>(out4);
  k_probs_check_init<<<1, 1, 0, st>>>(state);
  if (npix > 0) {
    int64_t b = (npix + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    k_probs_check<<<(unsigned)b, 256, 0, st>>>(probs, npix, num_classes, state);
  }
  k_probs_check_fin<<<1, 1, 0, st>>>(state);
  return check_launch("tfb_probs_check");
}

extern "C" int tfb_confusion(const int32_t *pred, const int32_t *ref, int64_t npix, int num_classes,
                             const uint8_t *ignore, unsigned long long *confusion, unsigned long long *unknown,
                             unsigned long long *valid_count, void *stream) {
  TFB_REQUIRE(pred && ref && confusion && unknown && valid_count, TFB_ERR_DATA, "tfb_confusion: null argument");
  TFB_REQUIRE(num_classes >= 1, TFB_ERR_VALUE, "num_classes must be >= 1");
  if (npix <= 0) return TFB_OK;
  int64_t b = (npix + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  k_confusion<<<(unsigned)b, 256, 0, static_cast<cudaStream_t>(stream)>>>(pred, ref, npix, num_classes, ignore,
                                                                          confusion, unknown, valid_count);
  return check_launch("tfb_confusion");
}

extern "C" int tfb_face_majority(const int32_t *texel_labels, const int32_t *steps, const int64_t *offsets,
                                 int64_t num_triangles, int num_classes, int32_t *face_class, void *stream) {
  TFB_REQUIRE(texel_labels && steps && offsets && face_class, TFB_ERR_DATA, "tfb_face_majority: null argument");
  TFB_REQUIRE(num_classes >= 1 && num_classes <= 6144, TFB_ERR_VALUE,
              "tfb_face_majority: num_classes %d outside 1..6144", num_classes);
  if (num_triangles <= 0) return TFB_OK;
  const size_t smem = (size_t)8 * num_classes * sizeof(unsigned int);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_face_majority, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t b = (num_triangles + 7) / 8;
  if (b > 148 * 8) b = 148 * 8;
  k_face_majority<<<(unsigned)b, 256, smem, static_cast<cudaStream_t>(stream)>>>(texel_labels, steps, offsets,
                                                                                 num_triangles, num_classes,
                                                                                 face_class);
  return check_launch("tfb_face_majority");
}
