// Fusion scatter-add (fusion.py:114-183) and its per-frame helpers.
//
// k_fuse is the HBM-bound hot kernel.  Work item = (frame, 32-pixel chunk):
// the chunk's (32, c) float32 probability rows are one contiguous span of the
// (H, W, c) map.  Every warp is an independent pipeline (no CTA barriers):
// lane 0 streams its items into a private shared-memory ring of NS stages
// with the Blackwell bulk-copy engine (cp.async.bulk … mbarrier::complete_tx,
// L2 evict_first: each probability byte is read once and must not evict the
// accumulator, which stays L2-resident at the BASELINE sizes), while the
// warp's lanes
//   1. hold the chunk's texel rows and weights in registers, prefetched one
//      and two items ahead (rows, then the dependent hit-count gather);
//   2. find runs of consecutive pixels on the same texel with ballots and cut
//      them into pieces at pixel-group starts (and every 4 pixels for the
//      product rule, 5 in k_fuse_fast); ~2.5 pixels per run at the BASELINE
//      scene;
//   3. work as lanes = (pixel group g, class quad q): each lane folds its
//      group's pixels of quad q straight out of the staged shared-memory rows
//      (sum, or product of <= 4 (5) clipped probabilities, f32x2 multiplies)
//      and lands every finished piece with ONE red.global.add.v4.f32, plus one
//      u32 count add per run of equal rows (by its head lane).
// Weights derived from the hit counts (pixels_iid / images_iid / blend) are
// equal inside a run, so w is applied once per item, and for the product
// rule sum_i w*log(p_i) is evaluated as w*log(prod_i p_i) over up to four
// pixels, with a MUFU lg2 log that switches to a log1p series above 0.9 so the
// relative accuracy holds as p -> 1.
// The float64 parity mode instead follows the reference arithmetic pixel by
// pixel (w*log(p) in double, fusion.py:177).  The per-pixel network argmax
// (render fallback, cli.py:293) is emitted from the same staged bytes.
#include <math.h>

#include <atomic>
#include <mutex>

#include "common.cuh"
#include "log_f64.cuh"

#ifndef TFB_LOG_F64
#define TFB_LOG_F64 1  // float64 logs through the table-driven tfb_log::log_f64 (else libdevice log)
#endif

namespace tfb {
namespace {

#ifndef TFB_FUSE_WARPS
#define TFB_FUSE_WARPS 8
#endif
#ifndef TFB_FUSE_REPACK
#define TFB_FUSE_REPACK 0  // 1: compile-time c % 4 != 0 scans a 16-byte-quad repack of each stage (measured slower)
#endif
#ifndef TFB_FUSE_NS_SHALLOW
#define TFB_FUSE_NS_SHALLOW 1
#endif
#ifndef TFB_FUSE_NS
#define TFB_FUSE_NS 2
#endif
constexpr int kWarps = TFB_FUSE_WARPS;  // warps per CTA (independent pipelines)
#ifndef TFB_FUSE_CSPEC
#define TFB_FUSE_CSPEC 1
#endif
#ifndef TFB_PIECE
#ifndef TFB_FUSE_FOLDBUF
#define TFB_FUSE_FOLDBUF 1  // k_fuse_fast, compile-time c % 4 != 0: folded pieces through an aligned buffer (16-byte STS / LDS)
#endif
#ifndef TFB_ARGMAX_FAST
#define TFB_ARGMAX_FAST 1  // network argmax / pixel max: strict-greater pass, exact NaN pass only when needed
#endif
#ifndef TFB_FUSE_D64
#define TFB_FUSE_D64 1  // float64 accumulator (count-derived weights, c <= 128) through k_fuse_fast's D64 mode (else k_fuse<double>)
#endif
#ifndef TFB_FIX_TRANSPOSE
#define TFB_FIX_TRANSPOSE 1  // k_fuse_fast fixed-point epilogue: lanes take classes qi0 + k*QW (coalesced 64-bit adds)
#endif
#ifndef TFB_QUAD_CSPEC
#define TFB_QUAD_CSPEC 1  // k_fuse_fast: masked quads of a compile-time c % 4 != 0 read as 4 words + selects
#endif
#ifndef TFB_NEAR1_PACKED_C
#define TFB_NEAR1_PACKED_C 32  // k_fuse_fast: compile-time class counts below this evaluate the near-1 series branch-free
#endif
#define TFB_PIECE 5  // k_fuse_fast product pieces: 5 clipped values >= 1e-7 multiply to >= 1e-35, a normal float
#endif
constexpr int kChunk = 32;       // pixels per work item = one per lane
constexpr int kMaxFrames = 256;  // frames per launch (pointers travel in the kernel parameters, 2 KB)

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
  float wa, wb;  // k_fuse_fast: w = wa + wb / hits (pixels_iid 1,0; images_iid 0,1; blend 1-alpha,alpha)
  void *accum;
  int64_t stride;
  uint32_t *counts;
  int32_t *fallback;
  int NS;
  int64_t cpf;     // chunks per frame
  int64_t nitems;  // nframes * cpf
  // optional item order (tfb_fuse_order): items as (frame << 24 | chunk), sorted by the
  // accumulator row block they touch; *norder of them (empty chunks are left out)
  const uint32_t *order;
  const uint32_t *norder;
};

struct Geo {
  int nq;    // class quads
  int QW;    // quads handled per pass (<= 32)
  int G;     // pixel groups per warp (lanes = G x QW)
  int span;  // pixels per group
};

__host__ __device__ inline Geo geo_of(int c) {
  Geo g;
  g.nq = (c + 3) >> 2;
  g.QW = g.nq < 32 ? g.nq : 32;
  g.G = 32 / g.QW;
  g.span = (kChunk + g.G - 1) / g.G;
  return g;
}

struct WarpSmem {
  size_t stage_floats;  // per stage, multiple of 4
  size_t o_w, o_doff, o_max, o_bar, total;
};

__host__ __device__ inline size_t al(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline WarpSmem warp_layout(int c, int NS, int accbytes) {
  WarpSmem s;
  s.stage_floats = al((size_t)kChunk * c, 4);
  size_t o = (size_t)NS * s.stage_floats * 4;
  s.o_doff = o;
  o += (size_t)kChunk * 4;
  s.o_w = o = al(o, 16);
  o += (size_t)kChunk * accbytes;
  s.o_max = o;
  o += kChunk * 4;
  s.o_bar = o = al(o, 16);
  o += (size_t)NS * 8;
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

// np.clip(p, 1e-7, 1) with NaN passing through (fusion.py:177): NaN-propagating min/max
__device__ __forceinline__ float clip_mul(float x) {
  float y;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(y) : "f"(x), "f"(kMulClampF));
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(y) : "f"(y), "f"(1.0f));
  return y;
}

// np.clip((double)v, 1e-7, 1) for a float32 v, compared in float: no float lies in
// [1e-7, kMulClampF) (kMulClampF is the float just above 1e-7), so v < 1e-7 as a double
// exactly when v < kMulClampF.  NaN fails every comparison and passes through.
__device__ __forceinline__ double clip_mul64(float v) {
  return v < kMulClampF ? kMulClamp : (v > 1.0f ? 1.0 : (double)v);
}



__device__ __forceinline__ bool tma_ok(const float *src, int npix, int c) {
  const size_t bytes = (size_t)npix * c * 4;
  return (bytes % 16 == 0) && (((uintptr_t)src & 15) == 0) && bytes > 0;
}

// (frame, chunk) of a work item, advanced by the warp-grid stride without divisions;
// i is the item's index in the launch's item order when there is one
struct Pos {
  int f, ch, i;
};

__device__ __forceinline__ void advance(Pos &q, int dF, int dC, int cpf) {
  q.ch += dC;
  q.f += dF;
  if (q.ch >= cpf) {
    q.ch -= cpf;
    ++q.f;
  }
}

// The warp-grid walk over a launch's items: frame-major (ORD = false), or through the
// row-block order of tfb_fuse_order (ORD = true), which keeps the accumulator rows the
// in-flight items touch inside L2 when the whole accumulator does not fit.
template <bool ORD>
struct Walk {
  int dF, dC, cpf, GW, n, nframes;
  const uint32_t *order;
  __device__ __forceinline__ Pos at(int i) const {
    if (i >= n) return Pos{nframes, 0, i};
    const uint32_t it = __ldg(order + i);
    return Pos{(int)(it >> 24), (int)(it & 0xffffffu), i};
  }
  __device__ __forceinline__ Pos first(int gw) const { return ORD ? at(gw) : Pos{gw / cpf, gw % cpf, gw}; }
  __device__ __forceinline__ void next(Pos &q) const {
    if (ORD) q = at(q.i + GW);
    else advance(q, dF, dC, cpf);
  }
};

__device__ __forceinline__ int32_t row_at(const FuseParams &p, Pos q, int lane) {
  if (q.f >= p.nframes) return -1;
  const int pix = q.ch * kChunk + lane;
  return pix < (int)p.hw ? __ldg(p.rows + (q.f * (int)p.hw + pix)) : -1;
}

// raw weight source (hit count bits or explicit weight), loaded one item ahead
// and converted only when used, so the gather latency overlaps a whole item
__device__ __forceinline__ double wsrc_at(const FuseParams &p, Pos q, int lane, int32_t r) {
  if (r < 0 || q.f >= p.nframes || p.wmode == TFB_W_PIXELS_IID) return 0.0;
  if (p.wmode == TFB_W_EXPLICIT) return __ldg(p.weights + (q.f * (int)p.hw + q.ch * kChunk + lane));
  return __longlong_as_double((long long)__ldg(p.hits + ((int64_t)q.f * p.n_x + r)));
}

// fusion.py:132-141
template <typename AccT>
__device__ __forceinline__ AccT weight_from(const FuseParams &p, double src, int32_t r) {
  if (r < 0) return (AccT)0;
  if (p.wmode == TFB_W_PIXELS_IID) return (AccT)1;
  if (p.wmode == TFB_W_EXPLICIT) return (AccT)src;
  const AccT per_image = (AccT)1 / (AccT)(uint32_t)__double_as_longlong(src);
  return p.wmode == TFB_W_IMAGES_IID ? per_image : ((AccT)1 - (AccT)p.alpha) + (AccT)p.alpha * per_image;
}

// log of a (product of) clipped probabilities, x in [1e-28, 1]: MUFU lg2 (2 ulp
// below 1/2, 2^-22.6 absolute above: at most 5.4e-6 relative for x <= 0.98, where
// |log2 x| >= 0.029).  Above kNear1 that absolute error would be large relative to
// |log x|, so the log1p series in t = x - 1 (exact) is used instead: |t| < 0.02,
// truncation t^5/5 below 3.2e-8 relative.  In log4 the series runs behind a warp
// vote, so warps with no such value skip it.
constexpr float kNear1 = 0.98f;
__device__ __forceinline__ float lg2_ln(float x) {
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
  return l * 0.693147180559945f;
}

__device__ __forceinline__ float log1p_series(float x) {
  const float t = x - 1.0f;
  return t * fmaf(t, fmaf(t, fmaf(t, -0.25f, 1.0f / 3.0f), -0.5f), 1.0f);
}

__device__ __forceinline__ void log4(float &a0, float &a1, float &a2, float &a3) {
  const float x0 = a0, x1 = a1, x2 = a2, x3 = a3;
  a0 = lg2_ln(x0);
  a1 = lg2_ln(x1);
  a2 = lg2_ln(x2);
  a3 = lg2_ln(x3);
  const bool near1 = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3)) > kNear1;
  if (__any_sync(__activemask(), near1)) {
    if (x0 > kNear1) a0 = log1p_series(x0);
    if (x1 > kNear1) a1 = log1p_series(x1);
    if (x2 > kNear1) a2 = log1p_series(x2);
    if (x3 > kNear1) a3 = log1p_series(x3);
  }
}

__device__ __forceinline__ float log_prob(float x) { return x > kNear1 ? log1p_series(x) : lg2_ln(x); }

// packed float32x2 multiply (sm_100 FMUL2)
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long ra = *reinterpret_cast<unsigned long long *>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long *>(&b);
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
  return *reinterpret_cast<float2 *>(&r);
}

// fixed-point accumulator element (TFB_ACCUM_FIXED): value * 2^32, round to nearest
__device__ __forceinline__ unsigned long long to_fixed(double x) {
  return (unsigned long long)__double2ll_rn(x * 4294967296.0);
}

// NumPy argmax / max of one pixel's c staged classes, in class order (first NaN wins,
// else the first maximum; cli.py:293, fusion.py:174).  Lanes hold different pixels, c
// words apart: with c % 4 == 0 the classes move as 16-byte quads (the 4c-byte pixel
// stride puts the quads of 8 lanes on at most 2-way conflicting banks, where scalar
// reads at a stride of 40 words would be 8-way); an odd c is conflict-free as scalars.
__device__ __forceinline__ float2 add2(float2 a, float2 b);
template <bool VEC>
__device__ __forceinline__ void pixel_argmax(const float *pp, int c, float &best, int &bi) {
  if (VEC && TFB_ARGMAX_FAST) {
    // one strict-greater pass (the first maximum wins) with a float32x2 running sum that
    // turns NaN if any class is NaN (or for inf - inf); only then the exact pass below
    best = pp[0];
    bi = 0;
    float2 sum = make_float2(0.f, 0.f);
    for (int k = 0; k < c; k += 4) {
      const float4 v = *reinterpret_cast<const float4 *>(pp + k);
      sum = add2(sum, make_float2(v.x, v.y));
      sum = add2(sum, make_float2(v.z, v.w));
      if (v.x > best) { best = v.x; bi = k; }
      if (v.y > best) { best = v.y; bi = k + 1; }
      if (v.z > best) { best = v.z; bi = k + 2; }
      if (v.w > best) { best = v.w; bi = k + 3; }
    }
    if (!isnan(sum.x + sum.y)) return;
  }
  best = pp[0];
  bi = 0;
  auto take = [&](float v, int k) {
    if (!isnan(best) && (isnan(v) || v > best)) {
      best = v;
      bi = k;
    }
  };
  if (VEC) {  // 16-byte quads; a padded last quad's extra lanes are not classes
    for (int k = 0; k < c; k += 4) {
      const float4 v = *reinterpret_cast<const float4 *>(pp + k);
      take(v.x, k);
      if (k + 1 < c) take(v.y, k + 1);
      if (k + 2 < c) take(v.z, k + 2);
      if (k + 3 < c) take(v.w, k + 3);
    }
  } else {
    for (int k = 1; k < c; ++k) take(pp[k], k);
  }
}

template <typename AccT, int AGG, bool EQW, bool FIX = false>
__global__ void __launch_bounds__(kWarps * 32) k_fuse(const __grid_constant__ FuseParams p) {
  // product rule in float32 with weights constant per run: fold w*log(prod p)
  constexpr bool kProd = (AGG == TFB_AGG_MUL) && EQW && sizeof(AccT) == 4;
  constexpr bool kProd64 = (AGG == TFB_AGG_MUL) && EQW && sizeof(AccT) == 8;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the float64 log's reduction table, per CTA in shared memory (lanes index it divergently)
  __shared__ double2 s_logtab[sizeof(AccT) == 8 && TFB_LOG_F64 ? (1 << tfb_log::kLogBits) : 1];
  if (sizeof(AccT) == 8 && TFB_LOG_F64) {
    for (int t = threadIdx.x; t < (1 << tfb_log::kLogBits); t += blockDim.x) s_logtab[t] = tfb_log::kTable[t];
    __syncthreads();
  }
  auto log64 = [&](double x) -> double { return TFB_LOG_F64 ? tfb_log::log_f64(x, s_logtab) : log(x); };
  const int c = p.c, NS = p.NS;
  const Geo geo = geo_of(c);
  const WarpSmem L = warp_layout(c, NS, (int)sizeof(AccT));
  unsigned char *ws = smem + (size_t)warp * L.total;
  float *stages = reinterpret_cast<float *>(ws);
  int32_t *sdoff = reinterpret_cast<int32_t *>(ws + L.o_doff);
  AccT *sw = reinterpret_cast<AccT *>(ws + L.o_w);
  float *smax = reinterpret_cast<float *>(ws + L.o_max);
  uint64_t *bar = reinterpret_cast<uint64_t *>(ws + L.o_bar);
  const int nw = blockDim.x >> 5;  // warps per CTA (fewer when c needs large stages)
  const int GW = gridDim.x * nw;
  const int gw = blockIdx.x * nw + warp;
  const int cpf = (int)p.cpf;
  const int dF = GW / cpf, dC = GW - dF * cpf;

  uint64_t policy = 0;
  if (lane == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto issue = [&](Pos q, int s) {
    const int64_t start = (int64_t)q.ch * kChunk;
    const int npix = (int)min((int64_t)kChunk, p.hw - start);
    const float *src = p.probs[q.f] + start * c;
    if (tma_ok(src, npix, c)) {
      const uint32_t bytes = (uint32_t)((size_t)npix * c * 4);
      mbar_expect_tx(bar + s, bytes);
      bulk_g2s(stages + (size_t)s * L.stage_floats, src, bytes, bar + s, policy);
    }
  };
  Pos cur{gw / cpf, gw % cpf, gw};
  if (lane == 0) {
    Pos q = cur;
    for (int s = 0; s < NS && q.f < p.nframes; ++s) {
      issue(q, s);
      advance(q, dF, dC, cpf);
    }
  }
  Pos nxt = cur, nn = cur;
  advance(nxt, dF, dC, cpf);
  advance(nn, dF, dC, cpf);
  advance(nn, dF, dC, cpf);

  const bool vec_ok = (c & 3) == 0;
  const unsigned upto = (2u << lane) - 1u;  // lanes <= this one
  // lane -> (pixel group g, class quad qi) for phase A
  const int g = lane / geo.QW, qi0 = lane - g * geo.QW;
  const int i0 = g * geo.span;
  const int i1 = min(i0 + geo.span, kChunk);
  const bool grp_start = (lane % geo.span) == 0;  // lane as a pixel: first pixel of its group

  int32_t r_cur = row_at(p, cur, lane);
  double ws_cur = wsrc_at(p, cur, lane, r_cur);
  int32_t r_nxt = row_at(p, nxt, lane);
  uint32_t phase = 0;
  int s = 0;
  while (cur.f < p.nframes) {
    // software prefetch: weight sources one item ahead, rows two items ahead
    const double ws_nxt = wsrc_at(p, nxt, lane, r_nxt);
    const int32_t r_nn = row_at(p, nn, lane);

    const int64_t start = (int64_t)cur.ch * kChunk;
    const int npix = (int)min((int64_t)kChunk, p.hw - start);
    const float *src = p.probs[cur.f] + start * c;
    float *st = stages + (size_t)s * L.stage_floats;

    // pieces: runs of equal rows, split at group starts (and every 4 pixels for
    // the float32 product rule, so a piece's product of clipped probabilities
    // stays normal; a float64 product of up to 32 values >= 1e-7 cannot underflow)
    const AccT w = weight_from<AccT>(p, ws_cur, r_cur);
    const int32_t prev = __shfl_up_sync(0xffffffffu, r_cur, 1);
    const bool chg = lane == 0 || prev != r_cur || grp_start;
    const unsigned cmask = __ballot_sync(0xffffffffu, chg);
    bool pstart = chg;
    if (kProd) {
      const int rs = 31 - __clz(cmask & upto);
      pstart = ((lane - rs) & 3) == 0;
    }
    const unsigned smask = __ballot_sync(0xffffffffu, pstart);
    {  // counts (fusion.py:182): one add per run of equal rows in the chunk
      const bool rstart = lane == 0 || prev != r_cur;
      const unsigned rmask = __ballot_sync(0xffffffffu, rstart);
      if (rstart && r_cur >= 0) {
        const unsigned above = rmask & ~upto;
        atomicAdd(p.counts + r_cur, (uint32_t)((above ? __ffs(above) - 1 : kChunk) - lane));
      }
    }
    sdoff[lane] = r_cur >= 0 ? (int32_t)((int64_t)r_cur * p.stride) : -1;  // accumulator row offset
    sw[lane] = w;

    if (tma_ok(src, npix, c)) {
      mbar_wait(bar + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    } else {
      for (int i = lane; i < npix * c; i += 32) st[i] = src[i];
    }
    __syncwarp();

    // per-pixel maximum (maxsum, fusion.py:174) and network argmax fallback (cli.py:293)
    if (AGG == TFB_AGG_MAXSUM || p.fallback) {
      if (lane < npix) {
        float best;
        int bi;
        if (vec_ok) pixel_argmax<true>(st + (size_t)lane * c, c, best, bi);
        else pixel_argmax<false>(st + (size_t)lane * c, c, best, bi);
        smax[lane] = best;
        if (p.fallback) p.fallback[(int64_t)cur.f * p.hw + start + lane] = bi;
      }
      __syncwarp();
    }

    for (int qb = 0; qb < geo.nq; qb += geo.QW) {
      // lanes = (pixel group g, class quad q): each group scans its pixels in
      // order, folding them into the running value of their piece; when a piece
      // ends the lane lands its quad with one vector reduction (fusion.py:180-181)
      const int q = qb + qi0;
      if (g < geo.G && q < geo.nq) {
        const int k0 = q * 4;
        const float *pp = st + (size_t)i0 * c + k0;
        const float pad = AGG == TFB_AGG_MUL ? 1.0f : 0.0f;
        AccT a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        float2 m01 = make_float2(1.f, 1.f), m23 = make_float2(1.f, 1.f);
        double2 d01 = make_double2(1.0, 1.0), d23 = make_double2(1.0, 1.0);  // float64 products
        int32_t doff = -1;
        AccT wrun = 0;
        auto flush = [&]() {
          if (doff < 0) return;
          if (sizeof(AccT) == 4) {
            float b0, b1, b2, b3;
            if (kProd) {
              b0 = m01.x; b1 = m01.y; b2 = m23.x; b3 = m23.y;
              log4(b0, b1, b2, b3);
            } else {
              b0 = (float)a0; b1 = (float)a1; b2 = (float)a2; b3 = (float)a3;
            }
            if (EQW) {
              const float wv = (float)wrun;
              b0 *= wv; b1 *= wv; b2 *= wv; b3 *= wv;
            }
            if (!vec_ok) {  // padding columns receive exact zeros
              if (k0 + 1 >= c) b1 = 0.f;
              if (k0 + 2 >= c) b2 = 0.f;
              if (k0 + 3 >= c) b3 = 0.f;
            }
            float *dst = reinterpret_cast<float *>(p.accum) + doff + k0;
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(b0), "f"(b1), "f"(b2),
                         "f"(b3));
          } else {
            double *dst = reinterpret_cast<double *>(p.accum) + doff + k0;
            double v[4] = {(double)a0, (double)a1, (double)a2, (double)a3};
            if (kProd64) {  // w * log(prod of the piece's clipped values) = sum of w * log(p)
              const double wv = (double)wrun;
              v[0] = wv * log64(d01.x);
              v[1] = wv * log64(d01.y);
              v[2] = wv * log64(d23.x);
              v[3] = wv * log64(d23.y);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (k0 + k < c) {
                if (FIX)  // integer adds commute exactly: the sum is independent of the atomic order
                  atomicAdd(reinterpret_cast<unsigned long long *>(dst) + k, to_fixed(v[k]));
                else
                  atomicAdd(dst + k, v[k]);
              }
          }
        };
#pragma unroll 2
        for (int i = i0; i < i1; ++i, pp += c) {
          float v0, v1, v2, v3;
          if (vec_ok) {
            const float4 v = *reinterpret_cast<const float4 *>(pp);
            v0 = v.x; v1 = v.y; v2 = v.z; v3 = v.w;
          } else {
            v0 = pp[0];
            v1 = k0 + 1 < c ? pp[1] : pad;
            v2 = k0 + 2 < c ? pp[2] : pad;
            v3 = k0 + 3 < c ? pp[3] : pad;
          }
          if ((smask >> i) & 1u) {  // a new piece starts at pixel i
            flush();
            doff = sdoff[i];
            wrun = sw[i];
            a0 = a1 = a2 = a3 = (AccT)0;
            m01 = make_float2(1.f, 1.f);
            m23 = make_float2(1.f, 1.f);
            d01 = make_double2(1.0, 1.0);
            d23 = make_double2(1.0, 1.0);
          }
          if (kProd64) {
            // float64 parity mode, product rule with one weight per piece: the
            // clipped values multiply in double, one log per piece and class
            d01.x *= clip_mul64(v0);
            d01.y *= clip_mul64(v1);
            d23.x *= clip_mul64(v2);
            d23.y *= clip_mul64(v3);
          } else if (kProd) {
            m01 = mul2(m01, make_float2(clip_mul(v0), clip_mul(v1)));
            m23 = mul2(m23, make_float2(clip_mul(v2), clip_mul(v3)));
          } else if (sizeof(AccT) == 4) {
            const float wi = EQW ? 1.0f : (float)sw[i];
            float t0 = v0, t1 = v1, t2 = v2, t3 = v3;
            if (AGG == TFB_AGG_MAXSUM) {
              const float mx = smax[i];
              t0 = v0 == mx ? v0 : 0.f; t1 = v1 == mx ? v1 : 0.f; t2 = v2 == mx ? v2 : 0.f; t3 = v3 == mx ? v3 : 0.f;
            } else if (AGG == TFB_AGG_MUL) {
              t0 = log_prob(clip_mul(v0)); t1 = log_prob(clip_mul(v1));
              t2 = log_prob(clip_mul(v2)); t3 = log_prob(clip_mul(v3));
            }
            a0 = fmaf(wi, t0, (float)a0); a1 = fmaf(wi, t1, (float)a1);
            a2 = fmaf(wi, t2, (float)a2); a3 = fmaf(wi, t3, (float)a3);
          } else {
            // float64 parity mode: the reference's per-pixel w * f(p) (fusion.py:171-177)
            const double wi = (double)sw[i];
            const float vv[4] = {v0, v1, v2, v3};
            double tt[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (AGG == TFB_AGG_SUM) tt[k] = (double)vv[k];
              else if (AGG == TFB_AGG_MAXSUM) tt[k] = vv[k] == smax[i] ? (double)vv[k] : 0.0;
              else tt[k] = log64(clip_mul64(vv[k]));
            }
            a0 += wi * tt[0]; a1 += wi * tt[1]; a2 += wi * tt[2]; a3 += wi * tt[3];
          }
        }
        flush();
      }
    }
    // stage s, table and side arrays are free again: every lane orders its generic-proxy reads
    // of the stage before the async-proxy refill, then the warp converges
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      Pos ahead = cur;
      for (int k = 0; k < NS; ++k) advance(ahead, dF, dC, cpf);
      if (ahead.f < p.nframes) issue(ahead, s);
    }
    cur = nxt;
    nxt = nn;
    advance(nn, dF, dC, cpf);
    r_cur = r_nxt;
    ws_cur = ws_nxt;
    r_nxt = r_nn;
    s = (s + 1 == NS) ? 0 : s + 1;
  }
}

// ---------------------------------------------------------------------------
// k_fuse_fast: the float32-accumulator, count-derived-weight (pixels_iid /
// images_iid / blend) case with 16-byte-aligned maps -- the BASELINE
// workload (VEC: c % 4 == 0, quads move as 16-byte vectors; otherwise as
// masked scalars, the last quad padded with the fold identity).  Same pipeline as k_fuse, but the piece epilogue is taken out of
// the divergent pixel scan:
//   scan      lanes = (pixel group g, class quad q) fold their group's pixels
//             into per-piece values (product / sum) and write each finished
//             piece's quad IN PLACE over the piece's first pixel in the staged
//             rows (that lane has already consumed those 16 bytes);
//   epilogue  converged: lanes = (piece, quad) pairs read the folded quads back
//             and land w*log2(prod)*ln2 (or w*sum) with one red.v4 each; the
//             near-1 log correction runs behind a full-warp vote.
// The product rule clips lazily: the scan tracks min/max of the raw values
// (2 FMNMX3 per pixel for each) and recomputes a piece with np.clip semantics
// only when a value falls outside [1e-7, 1] (NaN propagates through the
// product unchanged, as through np.clip + np.log).
// ---------------------------------------------------------------------------
struct FastSmem {
  size_t stage_floats, o_pad, o_head, o_max, o_bar, total;
};

// cpad > 0: a per-warp working copy of the landed stage with the class stride padded
// to cpad (a multiple of 4), so c % 4 != 0 rows move as 16-byte quads
__host__ __device__ inline FastSmem fast_layout(int c, int NS, int cpad = 0) {
  FastSmem s;
  s.stage_floats = (size_t)kChunk * c;  // 128*c bytes: every stage starts 16-byte aligned
  size_t o = (size_t)NS * s.stage_floats * 4;
  s.o_pad = o;
  o += (size_t)kChunk * cpad * 4;
  s.o_head = o;  // int4 per valid piece: {accumulator offset, weight bits, first-pixel float offset, 0}
  o += (size_t)kChunk * 16;
  s.o_max = o;
  o += (size_t)kChunk * 4;
  s.o_bar = o = al(o, 16);
  o += (size_t)NS * 8;
  s.total = al(o, 128);
  return s;
}

__device__ __forceinline__ float lg2_approx(float x) {
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
  return l;
}

// log2(x) for x in (kNear1, 1] from the log1p series in t = x - 1 (exact), scaled by 1/ln2
__device__ __forceinline__ float log2_series(float x) {
  const float t = x - 1.0f;
  constexpr float k = 1.4426950408889634f;
  return t * fmaf(t, fmaf(t, fmaf(t, -k / 4.0f, k / 3.0f), -k / 2.0f), k);
}

// log2_series on two values at once (sm_100 packed f32x2 add / fma / mul): the same
// operations in the same order per element, so each result is bit-identical to log2_series
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long *>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long *>(&b);
  unsigned long long rc = *reinterpret_cast<unsigned long long *>(&c);
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2 *>(&r);
}

__device__ __forceinline__ float2 add2(float2 a, float2 b);
__device__ __forceinline__ float2 log2_series2(float2 x) {
  constexpr float k = 1.4426950408889634f;
  const float2 t = add2(x, make_float2(-1.0f, -1.0f));  // x - 1, exact (Sterbenz) as in log2_series
  float2 s = fma2(t, make_float2(-k / 4.0f, -k / 4.0f), make_float2(k / 3.0f, k / 3.0f));
  s = fma2(t, s, make_float2(-k / 2.0f, -k / 2.0f));
  s = fma2(t, s, make_float2(k, k));
  unsigned long long rt = *reinterpret_cast<const unsigned long long *>(&t);
  unsigned long long rs = *reinterpret_cast<unsigned long long *>(&s);
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(rt), "l"(rs));
  return *reinterpret_cast<float2 *>(&r);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long ra = *reinterpret_cast<unsigned long long *>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long *>(&b);
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
  return *reinterpret_cast<float2 *>(&r);
}

// quad access: 16-byte vectors when rows are 16-byte aligned (c % 4 == 0), else nv <= 4
// valid scalars with `pad` (the fold identity) in the missing lanes
// CC != 0 (compile-time c, c % 4 != 0): nv < 4 only on the last quad, where it is c % 4;
// the four words are read unconditionally (past a pixel's last class they are the next
// pixel's, or past the last stage the warp's head records: always inside the warp's shared
// memory) and the missing classes replaced by the pad with selects
template <bool VEC, int CC = 0>
__device__ __forceinline__ float4 lds4(const float *p, int nv, float pad) {
  if (VEC) return *reinterpret_cast<const float4 *>(p);
  if (CC != 0) {
    constexpr int t = CC % 4;
    float4 v = make_float4(p[0], p[1], p[2], p[3]);
    const bool last = t != 0 && nv < 4;
    if (t == 1) v.y = last ? pad : v.y;
    if (t == 1 || t == 2) v.z = last ? pad : v.z;
    v.w = last ? pad : v.w;
    return v;
  }
  return make_float4(p[0], nv > 1 ? p[1] : pad, nv > 2 ? p[2] : pad, nv > 3 ? p[3] : pad);
}

template <bool VEC>
__device__ __forceinline__ float4 ldg4(const float *p, int nv, float pad) {
  if (VEC) return __ldg(reinterpret_cast<const float4 *>(p));
  return make_float4(__ldg(p), nv > 1 ? __ldg(p + 1) : pad, nv > 2 ? __ldg(p + 2) : pad, nv > 3 ? __ldg(p + 3) : pad);
}

template <bool VEC, int CC = 0>
__device__ __forceinline__ void sts4(float *p, float4 v, int nv) {
  if (VEC) {
    *reinterpret_cast<float4 *>(p) = v;
    return;
  }
  if (CC != 0) {
    constexpr int t = CC % 4;
    const bool last = t != 0 && nv < 4;
    p[0] = v.x;
    if (t != 1 || !last) p[1] = v.y;
    if ((t != 1 && t != 2) || !last) p[2] = v.z;
    if (!last) p[3] = v.w;
    return;
  }
  p[0] = v.x;
  if (nv > 1) p[1] = v.y;
  if (nv > 2) p[2] = v.z;
  if (nv > 3) p[3] = v.w;
}

template <int AGG, bool VEC, int CC, bool ORD = false, bool FIX = false, bool D64 = false>
__global__ void __launch_bounds__(kWarps * 32) k_fuse_fast(const __grid_constant__ FuseParams p) {
  // D64: the float64 parity accumulator (fusion.py:171-177 in double): no scan; converged
  // epilogue lanes = (piece, class set) fold the piece's values in double straight from the
  // staged rows -- product of clipped values then w * log (mul), or the sum of w * p (sum;
  // maxsum keeps p only where it equals the pixel's max) -- and land them with float64 adds
  static_assert(!D64 || (!FIX && !ORD), "D64: float64 accumulator, frame-major walk");
  constexpr bool kProd = AGG == TFB_AGG_MUL;
  __shared__ double2 s_logtab[D64 && kProd ? (1 << tfb_log::kLogBits) : 1];
  if (D64 && kProd) {
    for (int t = threadIdx.x; t < (1 << tfb_log::kLogBits); t += blockDim.x) s_logtab[t] = tfb_log::kTable[t];
    __syncthreads();
  }
  // compile-time c below TFB_NEAR1_PACKED_C: the near-1 log series without the warp vote
  constexpr bool kNear1Packed = CC != 0 && CC < TFB_NEAR1_PACKED_C;
#define TFB_QUAD_CC (TFB_QUAD_CSPEC ? CC : 0)
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // CC != 0: the class count is a compile-time constant (address steps and the
  // quad geometry fold into immediates); 0: read from the parameters
  const int c = CC ? CC : p.c, NS = p.NS;
  // compile-time c % 4 != 0: each landed stage is repacked into a working copy with the
  // class stride padded to a multiple of 4 (pad lanes = the fold identity), so the scan
  // and the epilogue move 16-byte quads as for c % 4 == 0 (QV) instead of masked scalars
  constexpr bool kPad = !VEC && !D64 && TFB_FUSE_REPACK && CC != 0 && (CC % 4) != 0;
  constexpr bool QV = VEC || kPad;
  // compile-time c % 4 != 0 without the repack: the scan reads the staged rows as masked
  // scalars, but writes each finished piece's quads as 16-byte vectors into an aligned
  // per-warp fold buffer (class stride cs4), which the epilogue reads back as vectors --
  // half the shared-memory wavefronts of scalar words on those two passes
  constexpr bool kFold = !VEC && !kPad && !D64 && TFB_FUSE_FOLDBUF && CC != 0 && (CC % 4) != 0;
  constexpr int cs4 = (CC + 3) & ~3;
  const int cs = kPad ? ((CC + 3) & ~3) : c;  // class stride of the working rows
  const Geo geo = geo_of(c);
  const FastSmem L = fast_layout(c, NS, (kPad || kFold) ? cs4 : 0);
  unsigned char *ws = smem + (size_t)warp * L.total;
  float *stages = reinterpret_cast<float *>(ws);
  float *padrows = reinterpret_cast<float *>(ws + L.o_pad);
  int4 *shead = reinterpret_cast<int4 *>(ws + L.o_head);
  float *smax = reinterpret_cast<float *>(ws + L.o_max);
  uint64_t *bar = reinterpret_cast<uint64_t *>(ws + L.o_bar);
  const int nw = blockDim.x >> 5;  // warps per CTA (fewer when c needs large stages)
  const int GW = gridDim.x * nw;
  const int gw = blockIdx.x * nw + warp;
  const int cpf = (int)p.cpf, hw = (int)p.hw;
  const int dF = GW / cpf, dC = GW - dF * cpf;
  const float wa = p.wa, wb = p.wb;
  const Walk<ORD> wk{dF, dC, cpf, GW, ORD ? (int)*p.norder : 0, p.nframes, p.order};

  uint64_t policy = 0;
  if (lane == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto issue = [&](Pos q, int s) {
    const int start = q.ch * kChunk;
    const int npix = min(kChunk, hw - start);
    // the bulk copy moves whole 16-byte units; a partial last chunk's tail (< 16 B,
    // only when c % 4 != 0) is copied by the lanes after the wait
    const uint32_t bytes = (uint32_t)(npix * c * 4) & ~15u;
    mbar_expect_tx(bar + s, bytes);
    if (bytes)
      bulk_g2s(stages + (size_t)s * L.stage_floats, p.probs[q.f] + (size_t)start * c, bytes, bar + s, policy);
  };
  Pos cur = wk.first(gw);
  Pos ahead = cur;  // next item to stage
  for (int s = 0; s < NS && ahead.f < p.nframes; ++s) {
    if (lane == 0) issue(ahead, s);
    wk.next(ahead);
  }
  Pos nxt = cur, nn = cur;
  wk.next(nxt);
  nn = nxt;
  wk.next(nn);

  const unsigned upto = (2u << lane) - 1u;  // lanes <= this one
  const int g = lane / geo.QW, qi0 = lane - g * geo.QW;
  const int i0 = g * geo.span;
  const int i1 = min(i0 + geo.span, kChunk);
  const bool grp_start = (lane % geo.span) == 0;
  const bool scan_lane = g < geo.G;

  auto hits_at = [&](Pos q, int32_t r) -> uint32_t {
    if (r < 0 || q.f >= p.nframes || wb == 0.0f) return 1u;
    return __ldg(p.hits + ((int64_t)q.f * p.n_x + r));
  };
  int32_t r_cur = row_at(p, cur, lane);
  uint32_t n_cur = hits_at(cur, r_cur);
  int32_t r_nxt = row_at(p, nxt, lane);
  uint32_t phase = 0;
  int s = 0;
  while (cur.f < p.nframes) {
    const uint32_t n_nxt = hits_at(nxt, r_nxt);
    const int32_t r_nn = row_at(p, nn, lane);
    const int npix = min(kChunk, hw - cur.ch * kChunk);
    float *st = stages + (size_t)s * L.stage_floats;

    // pieces (as in k_fuse) and their head records: one per piece on a covered texel
    const float w = fmaf(wb, rcp_approx((float)n_cur), wa);  // fusion.py:132-141
    const int32_t prev = __shfl_up_sync(0xffffffffu, r_cur, 1);
    const bool chg = lane == 0 || prev != r_cur || grp_start;
    const unsigned cmask = __ballot_sync(0xffffffffu, chg);
    bool pstart = chg;
    if (kProd && !D64) {  // float64 products of <= 32 values >= 1e-7 stay normal: no cut
      const int rs = 31 - __clz(cmask & upto);
      pstart = (lane - rs) % TFB_PIECE == 0;
    }
    const unsigned smask = __ballot_sync(0xffffffffu, pstart);
    const bool valid = pstart && r_cur >= 0;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    // counts (fusion.py:182): one add per run of equal rows in the chunk, not per
    // piece (a large triangle's pixels would all hit one address piece by piece)
    const bool rstart = (lane == 0 || prev != r_cur);
    const unsigned rmask = __ballot_sync(0xffffffffu, rstart);
    if (rstart && r_cur >= 0) {
      const unsigned above = rmask & ~upto;
      atomicAdd(p.counts + r_cur, (uint32_t)((above ? __ffs(above) - 1 : kChunk) - lane));
    }
    if (valid) {
      if (D64) {
        // float64 weight exactly as weight_from<double> (fusion.py:132-141); the piece's
        // first pixel and length (up to the next piece start)
        const double per_image = 1.0 / (double)n_cur;
        const double w64 = p.wmode == TFB_W_IMAGES_IID ? per_image
                           : p.wmode == TFB_W_BLEND    ? (1.0 - p.alpha) + p.alpha * per_image
                                                       : 1.0;
        const unsigned after = smask & ~upto;
        const int len = (after ? __ffs(after) - 1 : kChunk) - lane;
        shead[__popc(vmask & (upto >> 1))] =
            make_int4(r_cur * (int)p.stride, __double2loint(w64), lane | (len << 8), __double2hiint(w64));
      } else {
        const float wv = kProd ? w * 0.693147180559945f : w;
        shead[__popc(vmask & (upto >> 1))] = make_int4(r_cur * (int)p.stride, __float_as_int(wv), lane * (kFold ? cs4 : cs), 0);
      }
    }
    const int npv = __popc(vmask);

    mbar_wait(bar + s, (phase >> s) & 1u);
    phase ^= 1u << s;
    if (!VEC) {
      const int nfl = npix * c, done = (nfl * 4 & ~15) / 4;
      const float *src = p.probs[cur.f] + (size_t)cur.ch * kChunk * c;
      for (int i = done + lane; i < nfl; i += 32) st[i] = src[i];
    }
    __syncwarp();
    float *wst = st;  // the rows the scan, the argmax and the epilogue read (stride cs)
    if (kPad) {
      // lane = pixel: its CC scalars at stride CC (odd CC: conflict-free), four-aligned
      // 16-byte stores at stride cs, the pad lanes set to the fold identity
      if (lane < npix) {
        const float *sp = st + lane * CC;
        float *dp = padrows + lane * cs;
        const float one = kProd ? 1.0f : 0.0f;
#pragma unroll
        for (int q = 0; q < (CC + 3) / 4; ++q) {
          const int k = 4 * q;
          *reinterpret_cast<float4 *>(dp + k) = make_float4(
              sp[k], k + 1 < CC ? sp[k + 1] : one, k + 2 < CC ? sp[k + 2] : one, k + 3 < CC ? sp[k + 3] : one);
        }
      }
      __syncwarp();
      wst = padrows;
    }

    if (AGG == TFB_AGG_MAXSUM || p.fallback) {  // fusion.py:174, cli.py:293
      if (lane < npix) {
        float best;
        int bi;
        pixel_argmax<QV>(wst + (size_t)lane * cs, c, best, bi);
        smax[lane] = best;
        if (p.fallback) p.fallback[(int64_t)cur.f * p.hw + cur.ch * kChunk + lane] = bi;
      }
      __syncwarp();
    }

    for (int qb = 0; qb < geo.nq; qb += geo.QW) {
      const int q = qb + qi0;
      const int nv = min(4, c - 4 * q);  // valid classes of this lane's quad
      const float one = kProd ? 1.0f : 0.0f;  // fold identity
      // ---- scan: fold each piece of this lane's group into its first pixel's slot.
      // Branch-free over the group's pixels: at a piece start the running value
      // is stored (one predicated STS.128) and reset by selects.
      // pixels past npix (a frame's partial last chunk) hold stale stage data: not scanned
      const int n = min(i1, npix) - i0;
      if (!D64 && scan_lane && q < geo.nq && vmask != 0u && n > 0) {
        const unsigned sm = smask >> i0;  // bit j: a piece starts at pixel i0 + j (bit 0 always set)
        float *pp = wst + (size_t)i0 * cs + 4 * q;
        // where finished pieces go: in place over the piece's first pixel, or its fold-buffer row
        float *pf = kFold ? padrows + (size_t)i0 * cs4 + 4 * q : pp;
        float *ps = pf;
        float4 v = lds4<QV, TFB_QUAD_CC>(pp, nv, one);
        if (AGG == TFB_AGG_MAXSUM) {
          const float mx = smax[i0];
          v.x = v.x == mx ? v.x : 0.f; v.y = v.y == mx ? v.y : 0.f;
          v.z = v.z == mx ? v.z : 0.f; v.w = v.w == mx ? v.w : 0.f;
        }
        float2 a01 = make_float2(v.x, v.y), a23 = make_float2(v.z, v.w);
        float mn01 = fminf(v.x, v.y), mn23 = fminf(v.z, v.w);
        float mx01 = fmaxf(v.x, v.y), mx23 = fmaxf(v.z, v.w);
        unsigned smr = sm >> 1;  // bit 0: does a piece start at the next pixel
#pragma unroll 2
        for (int j = 1; j < n; ++j) {
          pp += cs;
          if (kFold) pf += cs4;
          v = lds4<QV, TFB_QUAD_CC>(pp, nv, one);
          const bool start = smr & 1u;
          smr >>= 1;
          if (start) sts4<QV || kFold, TFB_QUAD_CC>(ps, make_float4(a01.x, a01.y, a23.x, a23.y), nv);
          ps = start ? (kFold ? pf : pp) : ps;
          a01.x = start ? one : a01.x; a01.y = start ? one : a01.y;
          a23.x = start ? one : a23.x; a23.y = start ? one : a23.y;
          if (kProd) {
            a01 = mul2(a01, make_float2(v.x, v.y));
            a23 = mul2(a23, make_float2(v.z, v.w));
            mn01 = fminf(fminf(mn01, v.x), v.y);
            mn23 = fminf(fminf(mn23, v.z), v.w);
            mx01 = fmaxf(fmaxf(mx01, v.x), v.y);
            mx23 = fmaxf(fmaxf(mx23, v.z), v.w);
          } else {
            if (AGG == TFB_AGG_MAXSUM) {
              const float mx = smax[i0 + j];
              v.x = v.x == mx ? v.x : 0.f; v.y = v.y == mx ? v.y : 0.f;
              v.z = v.z == mx ? v.z : 0.f; v.w = v.w == mx ? v.w : 0.f;
            }
            a01 = add2(a01, make_float2(v.x, v.y));
            a23 = add2(a23, make_float2(v.z, v.w));
          }
        }
        sts4<QV || kFold, TFB_QUAD_CC>(ps, make_float4(a01.x, a01.y, a23.x, a23.y), nv);
        if (kProd && (fminf(mn01, mn23) < kMulClampF || fmaxf(mx01, mx23) > 1.0f)) {
          // rare: a value outside [1e-7, 1] in this group -> redo its pieces with
          // np.clip(p, 1e-7, 1) (fusion.py:177) from the global copy (the staged
          // first-pixel slots are already overwritten)
          const float *g4 = p.probs[cur.f] + ((size_t)cur.ch * kChunk + i0) * c + 4 * q;
          pp = kFold ? padrows + (size_t)i0 * cs4 + 4 * q : wst + (size_t)i0 * cs + 4 * q;
          ps = pp;
          a01 = make_float2(1.f, 1.f);
          a23 = a01;
          for (int j = 0; j < n; ++j, pp += (kFold ? cs4 : cs), g4 += c) {
            const bool start = (sm >> j) & 1u;
            if (start && j > 0) {
              sts4<QV || kFold, TFB_QUAD_CC>(ps, make_float4(a01.x, a01.y, a23.x, a23.y), nv);
              ps = pp;
              a01 = make_float2(1.f, 1.f);
              a23 = a01;
            }
            const float4 u = ldg4<VEC>(g4, nv, 1.0f);
            a01 = mul2(a01, make_float2(clip_mul(u.x), clip_mul(u.y)));
            a23 = mul2(a23, make_float2(clip_mul(u.z), clip_mul(u.w)));
          }
          sts4<QV || kFold, TFB_QUAD_CC>(ps, make_float4(a01.x, a01.y, a23.x, a23.y), nv);
        }
      }
      __syncwarp();
      // ---- epilogue (converged): lanes = (piece, quad), one red.v4 per pair (fusion.py:180-181)
      float *accq = reinterpret_cast<float *>(p.accum) + 4 * q;
      const float *stq = (kFold ? padrows : wst) + 4 * q;
      const bool lane_ok = scan_lane && q < geo.nq;
      // fixed-point accumulator, one quad pass (c <= 128): the epilogue lane of quad slot qi0
      // takes the piece's classes qi0 + k*QW (k < 4) instead of 4*q .. 4*q + 3, so each of its
      // four scalar 64-bit adds has the QW lanes of a piece on consecutive words (3 sectors
      // for c = 40, not one sector per lane); every class still lands exactly once
      const bool kT = FIX && TFB_FIX_TRANSPOSE && geo.nq <= 32;
      int cl[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) cl[k] = qi0 + k * geo.QW;
      // with c % 4 == 0 (VEC) and one quad pass, QW = c / 4: all four classes exist
      auto has = [&](int k) { return VEC || cl[k] < c; };
      if (D64) {
        // lanes = (piece, classes qi0 + k*QW): the piece's clipped values multiply in double in
        // pixel order (as k_fuse's float64 mode), one table-driven log per piece and class
        // (fusion.py:177), the adds coalesced over a piece's consecutive classes (c <= 128)
        for (int P = g; P - g < npv; P += geo.G) {
          if (lane_ok && P < npv && !kProd) {
            // sum / maxsum: the reference's per-pixel w * f(p) summed in double (fusion.py:171-175)
            const int4 h = shead[P];
            const int p0 = h.z & 0xff;
            const float *row = wst + (size_t)p0 * cs;
            const double wv = __hiloint2double(h.w, h.y);
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
            for (int j = 0; j < (h.z >> 8); ++j, row += cs) {
              float x0 = row[cl[0]], x1 = has(1) ? row[cl[1]] : 0.f, x2 = has(2) ? row[cl[2]] : 0.f,
                    x3 = has(3) ? row[cl[3]] : 0.f;
              if (AGG == TFB_AGG_MAXSUM) {  // fusion.py:174: p where p equals the pixel's max
                const float mxp = smax[p0 + j];
                x0 = x0 == mxp ? x0 : 0.f; x1 = x1 == mxp ? x1 : 0.f;
                x2 = x2 == mxp ? x2 : 0.f; x3 = x3 == mxp ? x3 : 0.f;
              }
              d0 += wv * (double)x0;
              d1 += wv * (double)x1;
              d2 += wv * (double)x2;
              d3 += wv * (double)x3;
            }
            double *dr = reinterpret_cast<double *>(p.accum) + h.x;
            atomicAdd(dr + cl[0], d0);
            if (has(1)) atomicAdd(dr + cl[1], d1);
            if (has(2)) atomicAdd(dr + cl[2], d2);
            if (has(3)) atomicAdd(dr + cl[3], d3);
          } else if (lane_ok && P < npv) {
            const int4 h = shead[P];
            const float *row = wst + (size_t)(h.z & 0xff) * cs;
            // np.clip(p, 1e-7, 1) is lazy, as in the float32 scan: the raw values multiply
            // and their min / max are tracked; a piece holding a value outside [1e-7, 1]
            // is redone with clipping (NaN is ignored by fminf / fmaxf and passes through
            // the product exactly as through clip + log)
            double d0 = 1.0, d1 = 1.0, d2 = 1.0, d3 = 1.0;
            float mn = 1.0f, mx = 0.0f;
            const float pad1 = 1.0f;
            for (int j = h.z >> 8; j > 0; --j, row += cs) {
              const float x0 = row[cl[0]], x1 = has(1) ? row[cl[1]] : pad1, x2 = has(2) ? row[cl[2]] : pad1,
                          x3 = has(3) ? row[cl[3]] : pad1;
              d0 *= (double)x0;
              d1 *= (double)x1;
              d2 *= (double)x2;
              d3 *= (double)x3;
              mn = fminf(fminf(mn, x0), fminf(x1, fminf(x2, x3)));
              mx = fmaxf(fmaxf(mx, x0), fmaxf(x1, fmaxf(x2, x3)));
            }
            if (mn < kMulClampF || mx > 1.0f) {
              row = wst + (size_t)(h.z & 0xff) * cs;
              d0 = d1 = d2 = d3 = 1.0;
              for (int j = h.z >> 8; j > 0; --j, row += cs) {
                d0 *= clip_mul64(row[cl[0]]);
                if (has(1)) d1 *= clip_mul64(row[cl[1]]);
                if (has(2)) d2 *= clip_mul64(row[cl[2]]);
                if (has(3)) d3 *= clip_mul64(row[cl[3]]);
              }
            }
            const double wv = __hiloint2double(h.w, h.y);
            double *dr = reinterpret_cast<double *>(p.accum) + h.x;
            atomicAdd(dr + cl[0], wv * tfb_log::log_f64(d0, s_logtab));
            if (has(1)) atomicAdd(dr + cl[1], wv * tfb_log::log_f64(d1, s_logtab));
            if (has(2)) atomicAdd(dr + cl[2], wv * tfb_log::log_f64(d2, s_logtab));
            if (has(3)) atomicAdd(dr + cl[3], wv * tfb_log::log_f64(d3, s_logtab));
          }
        }
      } else {
        for (int P = g; P - g < npv; P += geo.G) {
          const bool ok = lane_ok && P < npv;
          int4 h = make_int4(0, 0, 0, 0);
          float4 m = make_float4(0.5f, 0.5f, 0.5f, 0.5f);  // idle lanes must not trip the near-1 vote
          if (ok) {
            h = shead[P];
            if (kT) {
              const float *row = (kFold ? padrows : wst) + h.z;
              m = make_float4(row[cl[0]], has(1) ? row[cl[1]] : one, has(2) ? row[cl[2]] : one,
                              has(3) ? row[cl[3]] : one);
            } else {
              m = lds4<QV || kFold, TFB_QUAD_CC>(stq + h.z, nv, one);
            }
          }
          float b0 = m.x, b1 = m.y, b2 = m.z, b3 = m.w;
          if (kProd) {
            b0 = lg2_approx(m.x);
            b1 = lg2_approx(m.y);
            b2 = lg2_approx(m.z);
            b3 = lg2_approx(m.w);
            if (kNear1Packed) {
              // small c and short pieces: some lane of nearly every warp holds a value above
              // kNear1, so the series runs branch-free, two values per instruction
              const float2 s01 = log2_series2(make_float2(m.x, m.y)), s23 = log2_series2(make_float2(m.z, m.w));
              b0 = m.x > kNear1 ? s01.x : b0;
              b1 = m.y > kNear1 ? s01.y : b1;
              b2 = m.z > kNear1 ? s23.x : b2;
              b3 = m.w > kNear1 ? s23.y : b3;
            } else if (__any_sync(0xffffffffu, fmaxf(fmaxf(m.x, m.y), fmaxf(m.z, m.w)) > kNear1)) {
              if (m.x > kNear1) b0 = log2_series(m.x);
              if (m.y > kNear1) b1 = log2_series(m.y);
              if (m.z > kNear1) b2 = log2_series(m.z);
              if (m.w > kNear1) b3 = log2_series(m.w);
            }
          }
          const float wv = __int_as_float(h.y);
          const float2 o01 = mul2(make_float2(b0, b1), make_float2(wv, wv));
          const float2 o23 = mul2(make_float2(b2, b3), make_float2(wv, wv));
          if (ok) {
            if (FIX && kT) {
              unsigned long long *dr = reinterpret_cast<unsigned long long *>(p.accum) + h.x;
              atomicAdd(dr + cl[0], to_fixed(o01.x));
              if (has(1)) atomicAdd(dr + cl[1], to_fixed(o01.y));
              if (has(2)) atomicAdd(dr + cl[2], to_fixed(o23.x));
              if (has(3)) atomicAdd(dr + cl[3], to_fixed(o23.y));
            } else if (FIX) {
              // fixed-point accumulator (TFB_ACCUM_FIXED): the piece's float32 value, rounded
              // once to 2^-32 units; integer adds make the sum independent of their order
              unsigned long long *dq = reinterpret_cast<unsigned long long *>(p.accum) + h.x + 4 * q;
              atomicAdd(dq, to_fixed(o01.x));
              if (nv > 1) atomicAdd(dq + 1, to_fixed(o01.y));
              if (nv > 2) atomicAdd(dq + 2, to_fixed(o23.x));
              if (nv > 3) atomicAdd(dq + 3, to_fixed(o23.y));
            } else {
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(accq + h.x), "f"(o01.x), "f"(o01.y),
                           "f"(o23.x), "f"(o23.y));
            }
          }
        }
      }  // D64 / float32 and fixed-point epilogues
      __syncwarp();
    }
    // stage s is free again.  Every lane read it and wrote folded quads into it through the
    // generic proxy: each orders those accesses before the async-proxy refill, then the warp
    // converges and one lane issues the bulk copy (the CUTLASS producer convention).
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (ahead.f < p.nframes) {
      if (lane == 0) issue(ahead, s);
      wk.next(ahead);
    }
    cur = nxt;
    nxt = nn;
    wk.next(nn);
    r_cur = r_nxt;
    n_cur = n_nxt;
    r_nxt = r_nn;
    s = (s + 1 == NS) ? 0 : s + 1;
  }
}

std::atomic<int> g_fuse_ctas_per_sm{0};  // 0 = as many as fit (tfb_set_option(TFB_OPT_FUSE_CTAS_PER_SM))
std::atomic<int> g_fuse_fast{1};         // tfb_set_option(TFB_OPT_FUSE_FAST): 0 routes everything through k_fuse


// Per-device launch configuration of one kernel (dynamic shared memory attribute,
// occupancy), computed once per device and size; entry points stay re-entrant.
constexpr int kMaxDevices = 64;
struct LaunchCache {
  std::mutex mu;
  size_t bytes[kMaxDevices] = {};
  int blocks_per_sm[kMaxDevices] = {};
  int num_sms[kMaxDevices] = {};
};

constexpr size_t kSmemBudget = 227 * 1024;

// warps per CTA: kWarps, fewer when that many staging rings do not fit in shared memory
inline int warps_for(size_t per_warp) {
  int nw = kWarps;
  while (nw > 1 && per_warp * nw > kSmemBudget) nw >>= 1;
  return nw;
}

template <typename Kern>
int launch_persistent(Kern kern, LaunchCache &lc, size_t per_warp, const FuseParams &p, cudaStream_t st) {
  const int nw = warps_for(per_warp);
  const size_t bytes = per_warp * nw;
  int dev = 0;
  cudaGetDevice(&dev);
  TFB_REQUIRE(dev >= 0 && dev < kMaxDevices, TFB_ERR_CUDA, "tfb_fuse: device ordinal %d out of range", dev);
  int per_sm, sms;
  {
    std::lock_guard<std::mutex> guard(lc.mu);
    if (lc.bytes[dev] != bytes) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
        return check_launch("tfb_fuse: shared memory configuration");
      cudaDeviceGetAttribute(&lc.num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lc.blocks_per_sm[dev], kern, nw * 32, bytes);
      if (lc.blocks_per_sm[dev] < 1) lc.blocks_per_sm[dev] = 1;
      lc.bytes[dev] = bytes;
    }
    per_sm = lc.blocks_per_sm[dev];
    sms = lc.num_sms[dev];
  }
  if (g_fuse_ctas_per_sm > 0 && g_fuse_ctas_per_sm < per_sm) per_sm = g_fuse_ctas_per_sm;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (p.nitems + nw - 1) / nw;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, nw * 32, bytes, st>>>(p);
  return check_launch("tfb_fuse");
}

template <typename AccT, int AGG, bool EQW, bool FIX = false>
int launch_fuse(const FuseParams &p, cudaStream_t st) {
  static LaunchCache lc;
  return launch_persistent(k_fuse<AccT, AGG, EQW, FIX>, lc, warp_layout(p.c, p.NS, (int)sizeof(AccT)).total, p, st);
}

template <int AGG, bool VEC, int CC = 0>
int launch_fuse_fast(const FuseParams &p, cudaStream_t st, bool fix, bool d64 = false) {
  if (d64) {  // float64 accumulator: no scan, no padded rows
    static LaunchCache lcd;
    return launch_persistent(k_fuse_fast<AGG, VEC, CC, false, false, true>, lcd, fast_layout(p.c, p.NS, 0).total, p,
                             st);
  }
  // the padded working rows of k_fuse_fast's compile-time c % 4 != 0 repack
  constexpr int kPadCs = (!VEC && (TFB_FUSE_REPACK || TFB_FUSE_FOLDBUF) && CC != 0 && CC % 4 != 0) ? ((CC + 3) & ~3) : 0;
  const size_t bytes = fast_layout(p.c, p.NS, kPadCs).total;
  if (fix) {
    static LaunchCache lcf;
    return launch_persistent(k_fuse_fast<AGG, VEC, CC, false, true>, lcf, bytes, p, st);
  }
  if (p.order) {
    static LaunchCache lco;
    return launch_persistent(k_fuse_fast<AGG, VEC, CC, true>, lco, bytes, p, st);
  }
  static LaunchCache lc;
  return launch_persistent(k_fuse_fast<AGG, VEC, CC>, lc, bytes, p, st);
}

// Common class counts get their own instantiation (NYU40, ScanNet 20,
// Cityscapes 19, NYU13): 3-4 % faster than the runtime-c kernel at c = 40.
template <int AGG>
int launch_fuse_fast_c(const FuseParams &p, bool vec, cudaStream_t st, bool fix, bool d64 = false) {
#if TFB_FUSE_CSPEC
  switch (p.c) {
    case 40: return launch_fuse_fast<AGG, true, 40>(p, st, fix, d64);
    case 20: return launch_fuse_fast<AGG, true, 20>(p, st, fix, d64);
    case 19: return launch_fuse_fast<AGG, false, 19>(p, st, fix, d64);
    case 13: return launch_fuse_fast<AGG, false, 13>(p, st, fix, d64);
    default: break;
  }
#endif
  return vec ? launch_fuse_fast<AGG, true>(p, st, fix, d64) : launch_fuse_fast<AGG, false>(p, st, fix, d64);
}

template <typename AccT, int AGG, bool FIX = false>
int launch_fuse_w(const FuseParams &p, cudaStream_t st) {
  return p.wmode == TFB_W_EXPLICIT ? launch_fuse<AccT, AGG, false, FIX>(p, st)
                                   : launch_fuse<AccT, AGG, true, FIX>(p, st);
}

// ---- item order for accumulators beyond L2 (tfb_fuse_order) ------------------------------
// key of item (f, ch) = accumulator row block (row >> shift) of its first covered pixel,
// -1 when no pixel of the chunk is covered.  One thread per item: pixel 0's row (one sector
// per item) decides for nearly every chunk; only chunks starting on an uncovered pixel scan
// on.  Consecutive items mostly share a key, so the histogram adds are warp-aggregated.
__global__ void k_item_keys(const int32_t *rows, int64_t hw, int cpf, int64_t nitems, int shift, int32_t *keys,
                            uint32_t *hist) {
  const int64_t item = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int32_t key = -1;
  if (item < nitems) {
    const int64_t f = item / cpf, ch = item - f * cpf;
    const int64_t p0 = ch * kChunk, n = min((int64_t)kChunk, hw - p0);
    const int32_t *r = rows + f * hw + p0;
    int32_t row = __ldg(r);
    for (int64_t k = 1; row < 0 && k < n; ++k) row = __ldg(r + k);
    key = row >= 0 ? (row >> shift) : -1;
    keys[item] = key;
  }
  const unsigned act = __ballot_sync(0xffffffffu, key >= 0);
  if (key >= 0) {
    const unsigned peers = __match_any_sync(act, key);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + key, (uint32_t)__popc(peers));
  }
}

// exclusive scan of the key histogram in place (one CTA), total item count to *n
__global__ void __launch_bounds__(1024) k_key_scan(uint32_t *hist, int64_t nkeys, uint32_t *n) {
  __shared__ uint32_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (nkeys + 1023) / 1024, lo = t * per, hi = min(nkeys, lo + per);
  uint32_t sum = 0;
  for (int64_t k = lo; k < hi; ++k) sum += hist[k];
  part[t] = sum;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {  // Hillis-Steele inclusive scan of the thread sums
    const uint32_t v = t >= d ? part[t - d] : 0u;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint32_t run = part[t] - sum;
  for (int64_t k = lo; k < hi; ++k) {
    const uint32_t h = hist[k];
    hist[k] = run;
    run += h;
  }
  if (t == 1023) *n = part[1023];
}

// every covered item to its key's next slot: order = items grouped by ascending key
// (warp-aggregated slot claims; the order inside a key is arbitrary -- the fold is a sum)
__global__ void k_key_scatter(const int32_t *keys, int64_t nitems, int cpf, uint32_t *cursor, uint32_t *order) {
  const int64_t item = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int32_t key = item < nitems ? keys[item] : -1;
  const unsigned act = __ballot_sync(0xffffffffu, key >= 0);
  if (key < 0) return;
  const unsigned peers = __match_any_sync(act, key);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(cursor + key, (uint32_t)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  const int64_t f = item / cpf, ch = item - f * cpf;
  order[base + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)(f << 24) | (uint32_t)ch;
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

extern "C" size_t tfb_fuse_order_workspace_bytes(int64_t hw, int nframes, int64_t total_texels, int shift) {
  const int64_t cpf = (hw + kChunk - 1) / kChunk;
  const int64_t nkeys = (total_texels >> shift) + 1;
  return (size_t)(cpf * nframes) * 4 + (size_t)nkeys * 4 + 256;
}

extern "C" int tfb_fuse_order(const int32_t *rows, int64_t hw, int nframes, int64_t total_texels, int shift,
                              void *workspace, size_t workspace_bytes, uint32_t *order_out, uint32_t *n_out,
                              void *stream) {
  TFB_REQUIRE(rows && workspace && order_out && n_out, TFB_ERR_DATA, "tfb_fuse_order: null argument");
  TFB_REQUIRE(shift >= 0 && shift < 31, TFB_ERR_VALUE, "tfb_fuse_order: bad row-block shift %d", shift);
  TFB_REQUIRE(nframes >= 0 && nframes <= kMaxFrames, TFB_ERR_DATA, "tfb_fuse_order: %d frames > %d per launch",
              nframes, kMaxFrames);
  TFB_REQUIRE(workspace_bytes >= tfb_fuse_order_workspace_bytes(hw, nframes, total_texels, shift), TFB_ERR_CAPACITY,
              "tfb_fuse_order: workspace too small");
  const int64_t cpf = (hw + kChunk - 1) / kChunk;
  TFB_REQUIRE(cpf < (1 << 24), TFB_ERR_CAPACITY, "tfb_fuse_order: %lld chunks per frame", (long long)cpf);
  const int64_t nitems = cpf * nframes, nkeys = (total_texels >> shift) + 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t *keys = static_cast<int32_t *>(workspace);
  uint32_t *hist = reinterpret_cast<uint32_t *>(static_cast<char *>(workspace) + ((nitems * 4 + 255) / 256) * 256);
  if (cudaMemsetAsync(hist, 0, (size_t)nkeys * 4, st) != cudaSuccess) return check_launch("tfb_fuse_order");
  if (nitems == 0) return cudaMemsetAsync(n_out, 0, 4, st) == cudaSuccess ? TFB_OK : check_launch("tfb_fuse_order");
  const unsigned blocks = (unsigned)((nitems + 255) / 256);
  k_item_keys<<<blocks, 256, 0, st>>>(rows, hw, (int)cpf, nitems, shift, keys, hist);
  k_key_scan<<<1, 1024, 0, st>>>(hist, nkeys, n_out);
  k_key_scatter<<<blocks, 256, 0, st>>>(keys, nitems, (int)cpf, hist, order_out);
  return check_launch("tfb_fuse_order");
}

extern "C" int tfb_fuse(const int32_t *rows, int64_t hw, int nframes, const float *const *probs, int num_classes,
                        const uint32_t *texel_hits, const double *weights, int64_t total_texels, int aggregator,
                        int weight_mode, double alpha, void *accum, int accum_kind, int64_t accum_stride,
                        uint32_t *counts, int32_t *fallback_out, void *stream) {
  return tfb_fuse_ordered(rows, hw, nframes, probs, num_classes, texel_hits, weights, total_texels, aggregator,
                          weight_mode, alpha, accum, accum_kind, accum_stride, counts, fallback_out, nullptr, nullptr,
                          stream);
}

extern "C" int tfb_fuse_ordered(const int32_t *rows, int64_t hw, int nframes, const float *const *probs,
                                int num_classes, const uint32_t *texel_hits, const double *weights,
                                int64_t total_texels, int aggregator, int weight_mode, double alpha, void *accum,
                                int accum_kind, int64_t accum_stride, uint32_t *counts, int32_t *fallback_out,
                                const uint32_t *item_order, const uint32_t *n_items, void *stream) {
  TFB_REQUIRE(accum_kind >= TFB_ACCUM_F32 && accum_kind <= TFB_ACCUM_FIXED, TFB_ERR_VALUE,
              "unknown accumulator kind %d", accum_kind);
  const bool wide = accum_kind != TFB_ACCUM_F32;  // 8-byte accumulator elements
  TFB_REQUIRE(aggregator >= 0 && aggregator <= 2, TFB_ERR_VALUE, "unknown aggregator id %d", aggregator);
  TFB_REQUIRE(weight_mode >= 0 && weight_mode <= 3, TFB_ERR_VALUE, "unknown weight mode id %d", weight_mode);
  TFB_REQUIRE(num_classes >= 1, TFB_ERR_VALUE, "num_classes must be >= 1");
  TFB_REQUIRE(rows && probs && accum && counts, TFB_ERR_DATA, "tfb_fuse: null rows, probs, accum or counts");
  TFB_REQUIRE(weight_mode != TFB_W_EXPLICIT || weights, TFB_ERR_DATA, "tfb_fuse: explicit weights missing");
  TFB_REQUIRE(weight_mode == TFB_W_EXPLICIT || weight_mode == TFB_W_PIXELS_IID || texel_hits, TFB_ERR_DATA,
              "tfb_fuse: weight mode needs per-frame texel hit counts");
  TFB_REQUIRE(accum_stride >= num_classes, TFB_ERR_DATA, "tfb_fuse: accum stride %lld < classes %d",
              (long long)accum_stride, num_classes);
  TFB_REQUIRE(wide || (accum_stride % 4 == 0 && ((uintptr_t)accum & 15) == 0), TFB_ERR_DATA,
              "tfb_fuse: float32 accumulator rows must be 16-byte aligned (stride multiple of 4)");
  if (nframes <= 0 || hw <= 0) return TFB_OK;
  TFB_REQUIRE(hw + kChunk < (1LL << 31), TFB_ERR_CAPACITY, "tfb_fuse: %lld pixels per frame is too many",
              (long long)hw);
  // frames per launch: the kernel indexes a launch's pixels with 32-bit frame * hw + pixel
  int fpl = (int)(((1LL << 31) - 1) / (hw + kChunk));
  if (fpl > kMaxFrames) fpl = kMaxFrames;
  TFB_REQUIRE(total_texels * accum_stride < (1LL << 31), TFB_ERR_CAPACITY,
              "tfb_fuse: accumulator of %lld x %lld elements exceeds 32-bit row offsets", (long long)total_texels,
              (long long)accum_stride);
  const size_t stage = (size_t)kChunk * num_classes * 4;
  // staging depth per warp: small stages keep four in flight; otherwise one, so twice the
  // warps fit per SM (measured: cfg2 scatter -2 %, float64 -7 %), except where a warp needs
  // its own look-ahead -- the row-block item order walks items out of address order, and
  // the c % 4 != 0 kernel is issue-bound on few resident warps (2: configs[3] 20.7 -> 15.2
  // us/frame, configs[4] 46.2 -> 45.7)
  const bool deep = item_order != nullptr || num_classes % 4 != 0;
  const int NS = stage <= 2048 ? 4 : (deep ? TFB_FUSE_NS : TFB_FUSE_NS_SHALLOW);
  TFB_REQUIRE(warp_layout(num_classes, NS, wide ? 8 : 4).total <= kSmemBudget &&
                  fast_layout(num_classes, NS, (num_classes + 3) & ~3).total <= kSmemBudget,
              TFB_ERR_CAPACITY, "tfb_fuse: %d classes exceed the shared-memory staging budget of one warp",
              num_classes);
  FuseParams p;
  p.hw = hw;
  p.c = num_classes;
  p.hits = texel_hits;
  p.weights = weights;
  p.n_x = total_texels;
  p.wmode = weight_mode;
  p.alpha = alpha;
  p.wa = weight_mode == TFB_W_IMAGES_IID ? 0.0f : weight_mode == TFB_W_BLEND ? (float)(1.0 - alpha) : 1.0f;
  p.wb = weight_mode == TFB_W_IMAGES_IID ? 1.0f : weight_mode == TFB_W_BLEND ? (float)alpha : 0.0f;
  p.accum = accum;
  p.stride = accum_stride;
  p.counts = counts;
  p.NS = NS;
  p.cpf = (hw + kChunk - 1) / kChunk;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int f0 = 0; f0 < nframes; f0 += fpl) {
    const int nf = nframes - f0 < fpl ? nframes - f0 : fpl;
    for (int i = 0; i < kMaxFrames; ++i) p.probs[i] = i < nf ? probs[f0 + i] : nullptr;
    for (int i = 0; i < nf; ++i)
      TFB_REQUIRE(p.probs[i], TFB_ERR_DATA, "tfb_fuse: null probability pointer for frame %d", f0 + i);
    p.rows = rows + (int64_t)f0 * hw;
    p.weights = weights ? weights + (int64_t)f0 * hw : nullptr;
    p.hits = texel_hits ? texel_hits + (int64_t)f0 * total_texels : nullptr;
    p.fallback = fallback_out ? fallback_out + (int64_t)f0 * hw : nullptr;
    p.nframes = nf;
    p.nitems = p.cpf * nf;
    // the item order covers one launch and leaves out chunks with no covered pixel, so it is
    // used only when every item is in it or nothing per pixel is written (no fallback output)
    p.order = (item_order && nframes <= fpl && !fallback_out) ? item_order : nullptr;
    p.norder = p.order ? n_items : nullptr;
    // the specialised kernel serves float32 and fixed-point accumulators (the latter with
    // float32 piece arithmetic); float64 keeps the reference's per-pixel double arithmetic
    const bool fix = accum_kind == TFB_ACCUM_FIXED;
    bool fast = (!wide || fix) && weight_mode != TFB_W_EXPLICIT && g_fuse_fast;
    // float64 accumulator, product rule, count-derived weights, one class pass: k_fuse_fast's
    // D64 mode (the reference's float64 arithmetic per piece, converged epilogue)
    bool d64 = TFB_FUSE_D64 && accum_kind == TFB_ACCUM_F64 && weight_mode != TFB_W_EXPLICIT &&
               num_classes <= 128 && g_fuse_fast;
    for (int i = 0; i < nf && (fast || d64); ++i)
      if (((uintptr_t)p.probs[i] & 15) != 0) fast = d64 = false;
    const bool vec = num_classes % 4 == 0;
    int rc;
    if (fast) {
      switch (aggregator) {
        case TFB_AGG_SUM:
          rc = launch_fuse_fast_c<TFB_AGG_SUM>(p, vec, st, fix);
          break;
        case TFB_AGG_MAXSUM:
          rc = launch_fuse_fast_c<TFB_AGG_MAXSUM>(p, vec, st, fix);
          break;
        default:
          rc = launch_fuse_fast_c<TFB_AGG_MUL>(p, vec, st, fix);
          break;
      }
    } else if (d64) {
      switch (aggregator) {
        case TFB_AGG_SUM: rc = launch_fuse_fast_c<TFB_AGG_SUM>(p, vec, st, false, true); break;
        case TFB_AGG_MAXSUM: rc = launch_fuse_fast_c<TFB_AGG_MAXSUM>(p, vec, st, false, true); break;
        default: rc = launch_fuse_fast_c<TFB_AGG_MUL>(p, vec, st, false, true); break;
      }
    } else if (accum_kind == TFB_ACCUM_FIXED) {
      switch (aggregator) {
        case TFB_AGG_SUM: rc = launch_fuse_w<double, TFB_AGG_SUM, true>(p, st); break;
        case TFB_AGG_MAXSUM: rc = launch_fuse_w<double, TFB_AGG_MAXSUM, true>(p, st); break;
        default: rc = launch_fuse_w<double, TFB_AGG_MUL, true>(p, st); break;
      }
    } else if (wide) {
      switch (aggregator) {
        case TFB_AGG_SUM: rc = launch_fuse_w<double, TFB_AGG_SUM>(p, st); break;
        case TFB_AGG_MAXSUM: rc = launch_fuse_w<double, TFB_AGG_MAXSUM>(p, st); break;
        default: rc = launch_fuse_w<double, TFB_AGG_MUL>(p, st); break;
      }
    } else {
      switch (aggregator) {
        case TFB_AGG_SUM: rc = launch_fuse_w<float, TFB_AGG_SUM>(p, st); break;
        case TFB_AGG_MAXSUM: rc = launch_fuse_w<float, TFB_AGG_MAXSUM>(p, st); break;
        default: rc = launch_fuse_w<float, TFB_AGG_MUL>(p, st); break;
      }
    }
    if (rc != TFB_OK) return rc;
  }
  return TFB_OK;
}

extern "C" int tfb_set_option(int option, int value) {
  if (option == TFB_OPT_FUSE_CTAS_PER_SM) {
    TFB_REQUIRE(value >= 0, TFB_ERR_VALUE, "tfb_set_option: negative CTA cap");
    g_fuse_ctas_per_sm = value;
    return TFB_OK;
  }
  if (option == TFB_OPT_FUSE_FAST) {
    g_fuse_fast = value != 0;
    return TFB_OK;
  }
  set_error("tfb_set_option: unknown option %d", option);
  return TFB_ERR_VALUE;
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

namespace tfb {
namespace {
__global__ void k_test_log_f64(const double *x, double *y, int64_t n) {
  __shared__ double2 tab[1 << tfb_log::kLogBits];
  for (int t = threadIdx.x; t < (1 << tfb_log::kLogBits); t += blockDim.x) tab[t] = tfb_log::kTable[t];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = tfb_log::log_f64(x[i], tab);
}
}  // namespace
}  // namespace tfb

extern "C" int tfb_test_log_f64(const double *x, double *y, int64_t n, void *stream) {
  TFB_REQUIRE(n >= 0 && (n == 0 || (x && y)), TFB_ERR_DATA, "tfb_test_log_f64: bad arguments");
  if (n == 0) return TFB_OK;
  const int64_t blocks = (n + 255) / 256;
  tfb::k_test_log_f64<<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, y,
                                                                                                              n);
  return check_launch("tfb_test_log_f64");
}
