// Fusion scatter-add (fusion.py:114-183) and its per-frame helpers.
//
// k_fuse is the HBM-bound hot kernel.  It is persistent (grid = resident CTAs
// across the 148 SMs) and walks (frame, chunk) work items, a chunk being P
// consecutive pixels whose (P, c) float32 probability rows are one
// contiguous span of the (H, W, c) map.  One elected thread streams each
// chunk into a shared-memory ring of NS stages with the Blackwell bulk-copy
// engine (cp.async.bulk … mbarrier::complete_tx, L2 evict_first hint: each
// probability byte is read exactly once and must not evict the accumulator,
// which stays L2-resident at the BASELINE sizes).  While later chunks are in
// flight the CTA:
//   1. gathers each pixel's texel row and weight (pixels_iid / images_iid /
//      blend from the per-frame texel hit counts, or explicit weights);
//   2. finds runs of consecutive pixels on the same texel (segments; at the
//      BASELINE scene ~2.5 pixels per run along a scanline);
//   3. gives every thread (segment, 4-class quad) items: the run's weighted
//      transformed probabilities (w·p, w·p·[p==max], w·log clip(p)) are summed
//      from shared memory and land with ONE vector reduction
//      red.global.add.v4.f32 per quad, plus one u32 count add per run.
// The per-pixel network argmax used as the render fallback (cli.py:293,
// bindings/__init__.py:112) is emitted from the same staged bytes when asked.
#include <math.h>

#include "common.cuh"

namespace tfb {
namespace {

constexpr int kFuseThreads = 256;
constexpr int kMaxFrames = 32;  // frames per launch (pointers travel in the kernel parameters)

struct FuseParams {
  const float *probs[kMaxFrames];
  const int32_t *rows;
  int64_t hw;
  int nframes;
  int c;
  const uint32_t *hits;
  const double *weights;
  int64_t n_x;
  int wmode;
  double alpha;
  void *accum;
  int64_t stride;
  uint32_t *counts;
  int32_t *fallback;
  int P;
  int NS;
  int64_t cpf;     // chunks per frame
  int64_t nitems;  // nframes * cpf
};

struct Smem {
  size_t stage_floats;  // per stage, multiple of 4
  size_t o_row, o_w, o_max, o_head, o_len, o_bar, o_misc, total;
};

__host__ __device__ inline size_t al(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem smem_layout(int P, int c, int NS, int accbytes) {
  Smem s;
  s.stage_floats = al((size_t)P * c, 4);
  size_t o = (size_t)NS * s.stage_floats * 4;
  s.o_w = o = al(o, 16);
  o += (size_t)P * accbytes;
  s.o_row = o = al(o, 16);
  o += (size_t)P * 4;
  s.o_max = o = al(o, 16);
  o += (size_t)P * 4;
  s.o_head = o = al(o, 16);
  o += (size_t)P * 4;
  s.o_len = o = al(o, 16);
  o += (size_t)P * 4;
  s.o_bar = o = al(o, 16);
  o += (size_t)NS * 8;
  s.o_misc = o = al(o, 16);
  o += 64;
  s.total = al(o, 128);
  return s;
}

__device__ __forceinline__ uint32_t sptr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(sptr(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sptr(dst)),
      "l"(src), "r"(bytes), "r"(sptr(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ float np_clipf(float x, float lo, float hi) {
  // NumPy clip kernel semantics: MIN(MAX(x, lo), hi), NaN passes through
  if (isnan(x)) return x;
  x = x > lo ? x : lo;
  return x < hi ? x : hi;
}

__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
  if (isnan(x)) return x;
  x = x > lo ? x : lo;
  return x < hi ? x : hi;
}

template <int AGG>
__device__ __forceinline__ float xf_f(float v, float mx) {
  if (AGG == TFB_AGG_SUM) return v;
  if (AGG == TFB_AGG_MAXSUM) return v == mx ? v : 0.0f;  // fusion.py:174-175 (ties kept)
  return logf(np_clipf(v, kMulClampF, 1.0f));            // fusion.py:177
}

template <int AGG>
__device__ __forceinline__ double xf_d(float v, float mx) {
  if (AGG == TFB_AGG_SUM) return (double)v;
  if (AGG == TFB_AGG_MAXSUM) return v == mx ? (double)v : 0.0;
  return log(np_clip((double)v, kMulClamp, 1.0));
}

__device__ __forceinline__ bool tma_ok(const float *src, int npix, int c) {
  const size_t bytes = (size_t)npix * c * 4;
  return (bytes % 16 == 0) && (((uintptr_t)src & 15) == 0) && bytes > 0;
}

template <typename AccT, int AGG>
__global__ void __launch_bounds__(kFuseThreads) k_fuse(const __grid_constant__ FuseParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int P = p.P, c = p.c, NS = p.NS;
  const Smem L = smem_layout(P, c, NS, (int)sizeof(AccT));
  float *stages = reinterpret_cast<float *>(smem);
  AccT *sw = reinterpret_cast<AccT *>(smem + L.o_w);
  int32_t *srow = reinterpret_cast<int32_t *>(smem + L.o_row);
  float *smax = reinterpret_cast<float *>(smem + L.o_max);
  int32_t *shead = reinterpret_cast<int32_t *>(smem + L.o_head);
  int32_t *slen = reinterpret_cast<int32_t *>(smem + L.o_len);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.o_bar);
  int32_t *misc = reinterpret_cast<int32_t *>(smem + L.o_misc);  // [0..7] warp counts, [8] nseg
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x;

  uint64_t policy = 0;
  if (tid == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int64_t item, int s) {
    const int64_t f = item / p.cpf, ch = item - f * p.cpf;
    const int64_t start = ch * P;
    const int npix = (int)min((int64_t)P, p.hw - start);
    const float *src = p.probs[f] + start * c;
    if (tma_ok(src, npix, c)) {
      const uint32_t bytes = (uint32_t)((size_t)npix * c * 4);
      mbar_expect_tx(bar + s, bytes);
      bulk_g2s(stages + (size_t)s * L.stage_floats, src, bytes, bar + s, policy);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      const int64_t item = blockIdx.x + (int64_t)s * G;
      if (item < p.nitems) issue(item, s);
    }
  }

  const int nq = (c + 3) >> 2;
  const bool vec_ok = (c & 3) == 0;
  uint32_t phase = 0;
  int64_t it = 0;
  for (int64_t item = blockIdx.x; item < p.nitems; item += G, ++it) {
    const int s = (int)(it % NS);
    const int64_t f = item / p.cpf, ch = item - f * p.cpf;
    const int64_t start = ch * P;
    const int npix = (int)min((int64_t)P, p.hw - start);
    const float *src = p.probs[f] + start * c;
    float *st = stages + (size_t)s * L.stage_floats;

    // (1) per-pixel texel row and weight (fusion.py:114-142, 167-169)
    if (tid < P) {
      int32_t r = -1;
      double w = 0.0;
      if (tid < npix) {
        r = p.rows[f * p.hw + start + tid];
        if (r >= 0) {
          if (p.wmode == TFB_W_EXPLICIT) {
            w = p.weights[f * p.hw + start + tid];
          } else if (p.wmode == TFB_W_PIXELS_IID) {
            w = 1.0;
          } else {
            const double per_image = 1.0 / (double)p.hits[f * p.n_x + r];
            w = p.wmode == TFB_W_IMAGES_IID ? per_image : (1.0 - p.alpha) + p.alpha * per_image;
          }
        }
      }
      srow[tid] = r;
      sw[tid] = (AccT)w;
    }
    if (tma_ok(src, npix, c)) {
      mbar_wait(bar + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    } else {
      for (int i = tid; i < npix * c; i += kFuseThreads) st[i] = src[i];
    }
    __syncthreads();

    // (2) per-pixel maximum (maxsum) and network argmax fallback
    if ((AGG == TFB_AGG_MAXSUM || p.fallback) && tid < npix) {
      const float *pp = st + (size_t)tid * c;
      float best = pp[0];
      int bi = 0;
      for (int k = 1; k < c; ++k) {
        const float v = pp[k];
        if (!isnan(best) && (isnan(v) || v > best)) {
          best = v;
          bi = k;
        }
      }
      smax[tid] = best;
      if (p.fallback) p.fallback[f * p.hw + start + tid] = bi;
    }
    // (3) segment heads: runs of equal rows
    bool head = false;
    if (tid < npix) {
      const int32_t r = srow[tid];
      head = r >= 0 && (tid == 0 || srow[tid - 1] != r);
    }
    const uint32_t hb = __ballot_sync(0xffffffffu, head);
    if (lane == 0) misc[warp] = __popc(hb);
    __syncthreads();
    if (head) {
      int base = 0;
      for (int w2 = 0; w2 < warp; ++w2) base += misc[w2];
      const int idx = base + __popc(hb & ((1u << lane) - 1u));
      const int32_t r = srow[tid];
      int len = 1;
      while (tid + len < npix && srow[tid + len] == r) ++len;
      shead[idx] = tid;
      slen[idx] = len;
    }
    if (tid == 0) {
      int n = 0;
      for (int w2 = 0; w2 < kFuseThreads / 32; ++w2) n += misc[w2];
      misc[8] = n;
    }
    __syncthreads();

    // (4) one vector reduction per (segment, class quad)
    const int nseg = misc[8];
    for (int q2 = tid; q2 < nseg * nq; q2 += kFuseThreads) {
      const int sg = q2 / nq;
      const int q = q2 - sg * nq;
      const int h = shead[sg], len = slen[sg];
      const int32_t r = srow[h];
      const int k0 = q * 4;
      if (sizeof(AccT) == 4) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        for (int i = h; i < h + len; ++i) {
          const float wv = (float)sw[i];
          const float mx = AGG == TFB_AGG_MAXSUM ? smax[i] : 0.f;
          const float *pp = st + (size_t)i * c + k0;
          float v0, v1, v2, v3;
          if (vec_ok) {
            const float4 v = *reinterpret_cast<const float4 *>(pp);
            v0 = v.x; v1 = v.y; v2 = v.z; v3 = v.w;
          } else {
            v0 = pp[0];
            v1 = k0 + 1 < c ? pp[1] : 1.0f;
            v2 = k0 + 2 < c ? pp[2] : 1.0f;
            v3 = k0 + 3 < c ? pp[3] : 1.0f;
          }
          a0 += wv * xf_f<AGG>(v0, mx);
          a1 += wv * xf_f<AGG>(v1, mx);
          a2 += wv * xf_f<AGG>(v2, mx);
          a3 += wv * xf_f<AGG>(v3, mx);
        }
        if (!vec_ok) {  // padding columns receive exact zeros
          if (k0 + 1 >= c) a1 = 0.f;
          if (k0 + 2 >= c) a2 = 0.f;
          if (k0 + 3 >= c) a3 = 0.f;
        }
        float *dst = reinterpret_cast<float *>(p.accum) + (int64_t)r * p.stride + k0;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a0), "f"(a1), "f"(a2),
                     "f"(a3)
                     : "memory");
      } else {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = h; i < h + len; ++i) {
          const double wv = (double)sw[i];
          const float mx = AGG == TFB_AGG_MAXSUM ? smax[i] : 0.f;
          const float *pp = st + (size_t)i * c + k0;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k0 + k < c) acc[k] += wv * xf_d<AGG>(pp[k], mx);
        }
        double *dst = reinterpret_cast<double *>(p.accum) + (int64_t)r * p.stride + k0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k0 + k < c) atomicAdd(dst + k, acc[k]);
      }
      if (q == 0) atomicAdd(p.counts + r, (uint32_t)len);
    }
    __syncthreads();  // stage s and the side arrays are free again
    if (tid == 0) {
      const int64_t nxt = item + (int64_t)NS * G;
      if (nxt < p.nitems) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nxt, s);
      }
    }
  }
}

template <typename AccT, int AGG>
int launch_fuse(const FuseParams &p, cudaStream_t st) {
  const Smem L = smem_layout(p.P, p.c, p.NS, (int)sizeof(AccT));
  auto kern = k_fuse<AccT, AGG>;
  static int configured_bytes = -1;
  static int blocks_per_sm = 0;
  static int num_sms = 0;
  if (configured_bytes != (int)L.total) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total) != cudaSuccess)
      return check_launch("tfb_fuse: shared memory configuration");
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kFuseThreads, L.total);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    configured_bytes = (int)L.total;
  }
  int64_t grid = (int64_t)num_sms * blocks_per_sm;
  if (grid > p.nitems) grid = p.nitems;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kFuseThreads, L.total, st>>>(p);
  return check_launch("tfb_fuse");
}

__global__ void k_rows_from_ids(const int32_t *tri, const int32_t *texel, int64_t npix, tfb_scene sc, int32_t *rows,
                                int32_t *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = tri[i];
    int32_t r = -1;
    if (t != -1) {
      const int32_t x = texel[i];
      if (t < 0 || t >= sc.num_triangles) {
        *bad = 1;
      } else {
        const int64_t s = sc.steps[t];
        if (x < 0 || x >= (s * s + s) / 2) *bad = 1;
        else r = (int32_t)(sc.offsets[t] + x);
      }
    }
    rows[i] = r;
  }
}

__global__ void k_count_hits(const int32_t *rows, int64_t hw, int64_t n_x, uint32_t *hits) {
  const int f = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[f * hw + i];
    if (r >= 0) {
      const unsigned act = __activemask();
      const unsigned peers = __match_any_sync(act, r);
      if ((int)(__ffs(peers) - 1) == (int)(threadIdx.x & 31))
        atomicAdd(hits + f * n_x + r, (uint32_t)__popc(peers));
    }
  }
}

__global__ void k_clear_hits(const int32_t *rows, int64_t hw, int64_t n_x, uint32_t *hits) {
  const int f = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[f * hw + i];
    if (r >= 0) hits[f * n_x + r] = 0u;
  }
}

__global__ void k_pixel_weights(const int32_t *rows, int64_t hw, const uint32_t *hits, int64_t n_x, int mode,
                                double alpha, double *out) {
  const int f = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[f * hw + i];
    double w = 0.0;
    if (r >= 0) {
      if (mode == TFB_W_PIXELS_IID) {
        w = 1.0;
      } else {
        const double per_image = 1.0 / (double)hits[f * n_x + r];
        w = mode == TFB_W_IMAGES_IID ? per_image : (1.0 - alpha) + alpha * per_image;
      }
    }
    out[f * hw + i] = w;
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 4096) b = 4096;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace
}  // namespace tfb

using namespace tfb;

extern "C" int tfb_fuse(const int32_t *rows, int64_t hw, int nframes, const float *const *probs, int num_classes,
                        const uint32_t *texel_hits, const double *weights, int64_t total_texels, int aggregator,
                        int weight_mode, double alpha, void *accum, int accum_is_f64, int64_t accum_stride,
                        uint32_t *counts, int32_t *fallback_out, void *stream) {
  TFB_REQUIRE(aggregator >= 0 && aggregator <= 2, TFB_ERR_VALUE, "unknown aggregator id %d", aggregator);
  TFB_REQUIRE(weight_mode >= 0 && weight_mode <= 3, TFB_ERR_VALUE, "unknown weight mode id %d", weight_mode);
  TFB_REQUIRE(num_classes >= 1, TFB_ERR_VALUE, "num_classes must be >= 1");
  TFB_REQUIRE(rows && probs && accum && counts, TFB_ERR_DATA, "tfb_fuse: null rows, probs, accum or counts");
  TFB_REQUIRE(weight_mode != TFB_W_EXPLICIT || weights, TFB_ERR_DATA, "tfb_fuse: explicit weights missing");
  TFB_REQUIRE(weight_mode == TFB_W_EXPLICIT || weight_mode == TFB_W_PIXELS_IID || texel_hits, TFB_ERR_DATA,
              "tfb_fuse: weight mode needs per-frame texel hit counts");
  TFB_REQUIRE(accum_stride >= num_classes, TFB_ERR_DATA, "tfb_fuse: accum stride %lld < classes %d",
              (long long)accum_stride, num_classes);
  TFB_REQUIRE(accum_is_f64 || (accum_stride % 4 == 0 && ((uintptr_t)accum & 15) == 0), TFB_ERR_DATA,
              "tfb_fuse: float32 accumulator rows must be 16-byte aligned (stride multiple of 4)");
  if (nframes <= 0 || hw <= 0) return TFB_OK;
  int P = 128;
  while (P > 8 && (size_t)P * num_classes * 4 > 48 * 1024) P >>= 1;
  TFB_REQUIRE((size_t)P * num_classes * 4 <= 96 * 1024, TFB_ERR_CAPACITY,
              "tfb_fuse: %d classes exceed the shared-memory staging budget", num_classes);
  const size_t stage = (size_t)P * num_classes * 4;
  int NS = (int)((96 * 1024) / (stage ? stage : 1));
  if (NS > 4) NS = 4;
  if (NS < 2) NS = 2;
  FuseParams p;
  p.hw = hw;
  p.c = num_classes;
  p.hits = texel_hits;
  p.weights = weights;
  p.n_x = total_texels;
  p.wmode = weight_mode;
  p.alpha = alpha;
  p.accum = accum;
  p.stride = accum_stride;
  p.counts = counts;
  p.P = P;
  p.NS = NS;
  p.cpf = (hw + P - 1) / P;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int f0 = 0; f0 < nframes; f0 += kMaxFrames) {
    const int nf = nframes - f0 < kMaxFrames ? nframes - f0 : kMaxFrames;
    for (int i = 0; i < kMaxFrames; ++i) p.probs[i] = i < nf ? probs[f0 + i] : nullptr;
    for (int i = 0; i < nf; ++i)
      TFB_REQUIRE(p.probs[i], TFB_ERR_DATA, "tfb_fuse: null probability pointer for frame %d", f0 + i);
    p.rows = rows + (int64_t)f0 * hw;
    p.weights = weights ? weights + (int64_t)f0 * hw : nullptr;
    p.hits = texel_hits ? texel_hits + (int64_t)f0 * total_texels : nullptr;
    p.fallback = fallback_out ? fallback_out + (int64_t)f0 * hw : nullptr;
    p.nframes = nf;
    p.nitems = p.cpf * nf;
    int rc;
    if (accum_is_f64) {
      switch (aggregator) {
        case TFB_AGG_SUM: rc = launch_fuse<double, TFB_AGG_SUM>(p, st); break;
        case TFB_AGG_MAXSUM: rc = launch_fuse<double, TFB_AGG_MAXSUM>(p, st); break;
        default: rc = launch_fuse<double, TFB_AGG_MUL>(p, st); break;
      }
    } else {
      switch (aggregator) {
        case TFB_AGG_SUM: rc = launch_fuse<float, TFB_AGG_SUM>(p, st); break;
        case TFB_AGG_MAXSUM: rc = launch_fuse<float, TFB_AGG_MAXSUM>(p, st); break;
        default: rc = launch_fuse<float, TFB_AGG_MUL>(p, st); break;
      }
    }
    if (rc != TFB_OK) return rc;
  }
  return TFB_OK;
}

extern "C" int tfb_rows_from_ids(const int32_t *tri, const int32_t *texel, int64_t npix, const tfb_scene *scene,
                                 int32_t *rows_out, int32_t *bad_flag, void *stream) {
  TFB_REQUIRE(scene && tri && texel && rows_out && bad_flag, TFB_ERR_DATA, "tfb_rows_from_ids: null argument");
  if (npix <= 0) return TFB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_rows_from_ids<<<grid_for(npix), 256, 0, st>>>(tri, texel, npix, *scene, rows_out, bad_flag);
  return check_launch("tfb_rows_from_ids");
}

extern "C" int tfb_count_hits(const int32_t *rows, int64_t hw, int nframes, int64_t total_texels, uint32_t *hits,
                              void *stream) {
  TFB_REQUIRE(rows && hits, TFB_ERR_DATA, "tfb_count_hits: null argument");
  if (nframes <= 0 || hw <= 0) return TFB_OK;
  k_count_hits<<<dim3(grid_for(hw), nframes), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, hw, total_texels,
                                                                                           hits);
  return check_launch("tfb_count_hits");
}

extern "C" int tfb_clear_hits(const int32_t *rows, int64_t hw, int nframes, int64_t total_texels, uint32_t *hits,
                              void *stream) {
  TFB_REQUIRE(rows && hits, TFB_ERR_DATA, "tfb_clear_hits: null argument");
  if (nframes <= 0 || hw <= 0) return TFB_OK;
  k_clear_hits<<<dim3(grid_for(hw), nframes), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, hw, total_texels,
                                                                                           hits);
  return check_launch("tfb_clear_hits");
}

extern "C" int tfb_pixel_weights(const int32_t *rows, int64_t hw, int nframes, const uint32_t *hits,
                                 int64_t total_texels, int weight_mode, double alpha, double *out, void *stream) {
  TFB_REQUIRE(weight_mode >= 0 && weight_mode <= 2, TFB_ERR_VALUE, "unknown weight mode id %d", weight_mode);
  TFB_REQUIRE(rows && out && (weight_mode == TFB_W_PIXELS_IID || hits), TFB_ERR_DATA,
              "tfb_pixel_weights: null argument");
  if (nframes <= 0 || hw <= 0) return TFB_OK;
  k_pixel_weights<<<dim3(grid_for(hw), nframes), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, hw, hits, total_texels, weight_mode, alpha, out);
  return check_launch("tfb_pixel_weights");
}
