// Tile-binned z-buffer rasterizer, bit-exact with rasterizer.py:93-202.
//
// Per batch of frames (one launch per stage, all frames at once):
//   k_verts  per (frame, vertex): camera transform, clip outcode.
//   k_cull   per (frame, triangle): outcode cull (rasterizer.py:111 and empty
//            bboxes), survivors compacted (unclipped ones from the front of
//            the frame's list, near-clipped ones from the back).
//   k_setup  per survivor: FMA-ordered world->camera transform (geometry.py:161,
//            SURVEY A1), near-plane clip + fan (rasterizer.py:62-82, 113-122),
//            projection, bbox, signed area, CCW reorder and edge ownership
//            (rasterizer.py:136-164).  Each (sub)triangle becomes a 96-byte
//            record (key 2t+sub) at a slot fixed by its survivor-list position
//            and is appended to the fixed-capacity bin of every tile its bbox
//            overlaps (unordered).
//   k_raster one CTA per 16x8 tile, one thread per pixel.  Records staged
//            field-major; pair-parallel float64 edge tests (ownership rule
//            rasterizer.py:85-90); each pixel folds its covering records in
//            ascending (triangle, sub) key order with the reference's exact
//            test `z > 0 && z < depth - 1e-9` (rasterizer.py:171) — the
//            reference's sequential ascending-index loop, including the
//            non-transitive tie chains a packed atomicMin cannot reproduce.
//            The winner's perspective-correct barycentrics, (u, v) and texel
//            id (rasterizer.py:177-196) are evaluated once, in the epilogue.
//   k_raster_big  tiles with more records than a CTA stages, or an
//            overflowed bin: multipass K-smallest fold, same semantics.
//
// Exactness: every float64 operation of the reference expression is issued
// as an explicit round-to-nearest intrinsic in the reference's order and this
// translation unit is compiled with -fmad=false, so no contraction changes a
// rounding.  Only the camera transform uses FMA, in the order OpenBLAS dgemm
// evaluates `points @ R.T + t`.
#include <math.h>

#include <mutex>

#include "common.cuh"
#include "exact_div.cuh"

namespace tfb {
namespace {

#ifndef TFB_TW
#define TFB_TW 16
#endif
#ifndef TFB_TH
#define TFB_TH 8
#endif
constexpr int kTW = TFB_TW, kTH = TFB_TH;  // raster tile (pixels); one k_raster thread per pixel
constexpr int kTP = kTW * kTH;             // k_raster threads = tile pixels = staged records per tile
constexpr int kThreads = 256;              // setup-side kernels
#ifndef TFB_SETUP_MINB
#define TFB_SETUP_MINB 4  // k_setup CTAs per SM the register budget must allow (64 regs)
#endif
#ifndef TFB_FIRST_FAST
#define TFB_FIRST_FAST 1
#endif
#ifndef TFB_FUSED_SETUP
#define TFB_FUSED_SETUP 1  // clustered scenes: k_ccsetup (cull + record setup + binning in one pass)
#endif
#ifndef TFB_RASTER_NT
#define TFB_RASTER_NT 64  // k_raster threads per tile (= staged record capacity); kTP: one tier
#endif
constexpr int kRasterNT = TFB_RASTER_NT;
#ifndef TFB_FAST_LO
#define TFB_FAST_LO 0  // 1: test max e_k <= 1e100 per pixel instead of bounding the record's coordinates
#endif
#ifndef TFB_KEEP_PE
#define TFB_KEEP_PE 0  // 1: keep a sole covering pair's edge values in shared memory (else recomputed)
#endif
#ifndef TFB_RASTER_MINB32
#define TFB_RASTER_MINB32 32  // k_raster<32> CTAs per SM (the per-SM CTA limit; 64 registers)
#endif
#ifndef TFB_RASTER_MINB1
#define TFB_RASTER_MINB1 20  // k_raster<64> CTAs per SM the register budget must allow (48 registers)
#endif
#ifndef TFB_RASTER_MINB
#define TFB_RASTER_MINB 12  // 128-thread tile CTAs per SM the register budget must allow (40 regs; 1 % faster than 56 on the furnished room despite spills)
#endif
static_assert(kTW % 8 == 0 && kTH % 4 == 0 && kTP >= 64 && kTP <= 256, "tile shape: 8x4-pixel warp blocks");
constexpr int kCand = 8;
constexpr uint32_t kNoKey = 0xffffffffu;

struct __align__(16) RecGeom {
  double xs[3], ys[3], zs[3], dX[3], dY[3], area2;
};
static_assert(sizeof(RecGeom) == 128, "record geometry is one 128-byte line");

struct __align__(16) RecMeta {
  int16_t x0, x1, y0, y1;  // clamped pixel bbox (rasterizer.py:141-146)
  int32_t off;             // offsets[t]: first global texel row of the triangle (n_x < 2^31)
  uint32_t flags;          // bits 0-2 edge accept, 3 reordered, 4 clipped, 5-6 uv origin,
                           // 7 fan sub-triangle, 16-31 subdivision steps
};
static_assert(sizeof(RecMeta) == 16, "record meta is 16 bytes");

// What k_setup stores per record: the projected, CCW-ordered vertices and the
// meta (96 B).  The edge deltas and |area2| are derived exactly again where a
// record is staged (expand()), which keeps the per-frame record traffic at 3/4
// of a 128-byte line.
struct __align__(16) RecStore {
  RecMeta meta;
  double xs[3], ys[3], zs[3];
  uint32_t key;  // 2t + sub: the reference's (triangle, fan) order; kNoKey for an unused slot
  uint32_t pad;
};
static_assert(sizeof(RecStore) == 96, "stored record is 96 bytes");

// RecMeta from the first two doubles of a RecStore loaded as double2s
__device__ __forceinline__ RecMeta unpack_meta(double lo, double hi) {
  const unsigned long long a = (unsigned long long)__double_as_longlong(lo);
  const unsigned long long b = (unsigned long long)__double_as_longlong(hi);
  RecMeta m;
  m.x0 = (int16_t)(a & 0xffffu);
  m.x1 = (int16_t)((a >> 16) & 0xffffu);
  m.y0 = (int16_t)((a >> 32) & 0xffffu);
  m.y1 = (int16_t)(a >> 48);
  m.off = (int32_t)(b & 0xffffffffu);
  m.flags = (uint32_t)(b >> 32);
  return m;
}

// dX[k] = xs[b] - xs[a], dY[k] = ys[b] - ys[a] (a = k+1, b = k+2 mod 3) exactly as
// build_record forms them; |area2| from the reordered vertices: the reorder swaps
// the two products of rasterizer.py:148, and RN(B - A) = -RN(A - B), so the
// magnitude is bit-identical to the unordered value build_record took fabs of.
__device__ __forceinline__ void expand_derived(const double xs[3], const double ys[3], double dX[3], double dY[3],
                                               double &area2) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    dX[k] = __dsub_rn(xs[b], xs[a]);
    dY[k] = __dsub_rn(ys[b], ys[a]);
  }
  area2 = fabs(__dsub_rn(__dmul_rn(__dsub_rn(xs[1], xs[0]), __dsub_rn(ys[2], ys[0])),
                         __dmul_rn(__dsub_rn(ys[1], ys[0]), __dsub_rn(xs[2], xs[0]))));
}

__device__ __forceinline__ RecGeom expand(const RecStore &r) {
  RecGeom g;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g.xs[k] = r.xs[k];
    g.ys[k] = r.ys[k];
    g.zs[k] = r.zs[k];
  }
  expand_derived(g.xs, g.ys, g.dX, g.dY, g.area2);
  return g;
}

struct Cam {
  double R[9], T[3], fx, fy, cx, cy;
};

struct Work {
  RecStore *rec;        // per frame (2m slots): survivor at cand index c -> slot c if unclipped, 2c + fan half if
                        // near-clipped; so records fill [0, nA) and [2(m - nB), 2m) densely
  uint4 *cand;          // per frame (m entries): cull survivors {t | near-clip << 31, v0, v1, v2}; unclipped ones
                        // from the front (count fcnt[4f+2]), near-clipped ones from the back (count fcnt[4f+3])
  uint8_t *vcode;       // per frame per vertex: clip outcode (k_verts)
  int64_t nv;
  uint32_t *fcnt;       // fcnt[1]: big-tile count
  uint32_t *tile_count; // per frame per tile
  uint32_t *list;
  uint32_t *big;  // (frame, tile) codes handed to k_raster_big; count in fcnt[1]
  uint32_t *tl;    // tier lists: [0, nframes x ntiles) tiles for the 64-thread tier, then the 128-thread tier
  uint32_t *tcnt;  // their counts
  int64_t tlcap;   // entries per tier list (nframes x ntiles)
  uint32_t *csurv;  // per frame: surviving cluster ids (count fcnt[4f]); ncl entries per frame
  int64_t ncl;
  int64_t rs;   // record slots per frame (2m)
  int64_t bincap;  // records per tile bin (list holds nframes x ntiles bins)
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// scene clusters accepted for m triangles (64 slots each; see tfb_scene)
int64_t max_clusters(int64_t m) { return 2 * ((m + 63) / 64) + 1; }

bool carve(void *ws, size_t ws_bytes, int64_t nv, int64_t m, int nframes, int ntiles, int64_t bincap, Work &w,
           size_t *need_out) {
  const int64_t rs = 2 * (m > 0 ? m : 1);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  size_t o_rec = take(sizeof(RecStore) * rs * nframes);
  size_t o_cand = take(sizeof(uint4) * (size_t)(rs / 2) * nframes);
  size_t o_vcode = take((size_t)(nv > 0 ? nv : 1) * nframes);
  size_t o_fcnt = take(sizeof(uint32_t) * 4 * (nframes + 1));
  size_t o_tc = take(sizeof(uint32_t) * ntiles * nframes);
  size_t o_list = take(sizeof(uint32_t) * (size_t)bincap * ntiles * nframes);
  size_t o_big = take(sizeof(uint32_t) * ntiles * nframes);
  size_t o_tl = take(sizeof(uint32_t) * 2 * ntiles * nframes);
  const int64_t ncl = max_clusters(m);
  size_t o_csurv = take(sizeof(uint32_t) * (size_t)ncl * nframes);
  if (need_out) *need_out = off;
  if (!ws || ws_bytes < off) return false;
  char *b = static_cast<char *>(ws);
  w.rec = reinterpret_cast<RecStore *>(b + o_rec);
  w.cand = reinterpret_cast<uint4 *>(b + o_cand);
  w.vcode = reinterpret_cast<uint8_t *>(b + o_vcode);
  w.nv = nv > 0 ? nv : 1;
  w.fcnt = reinterpret_cast<uint32_t *>(b + o_fcnt);
  w.tcnt = w.fcnt + 4 * (int64_t)nframes;
  w.tlcap = (int64_t)ntiles * nframes;
  w.tile_count = reinterpret_cast<uint32_t *>(b + o_tc);
  w.list = reinterpret_cast<uint32_t *>(b + o_list);
  w.big = reinterpret_cast<uint32_t *>(b + o_big);
  w.tl = reinterpret_cast<uint32_t *>(b + o_tl);
  w.csurv = reinterpret_cast<uint32_t *>(b + o_csurv);
  w.ncl = ncl;
  w.rs = rs;
  w.bincap = bincap;
  return true;
}

// Tile bin capacity: `pair_capacity` (record/tile pairs budgeted per frame)
// spread over the tiles, default 4 pairs per triangle, at least 512 per tile
// (a 16x8 tile of the BASELINE scene holds ~20-60).  A tile whose bin
// overflows is still rasterized exactly by k_raster_big's full scan.
int64_t bin_capacity(int64_t pair_capacity, int64_t m, int ntiles) {
  int64_t c;
  if (pair_capacity > 0) {
    c = (pair_capacity + ntiles - 1) / ntiles;
  } else {
    c = (4 * m + ntiles - 1) / ntiles;
    if (c < 512) c = 512;
  }
  if (c < 1) c = 1;
  if (c > 0x7fffffffLL / (ntiles > 0 ? ntiles : 1)) c = 0x7fffffffLL / (ntiles > 0 ? ntiles : 1);
  return c;
}

__device__ __forceinline__ void load_cam(Cam &cam, const double *cams, int f) {
  double *d = reinterpret_cast<double *>(&cam);
  if (threadIdx.x < 16) d[threadIdx.x] = cams[(int64_t)f * 16 + threadIdx.x];
}

// geometry.py:159-161 through OpenBLAS dgemm: fma(z,R2,fma(y,R1,x*R0)) + t
__device__ __forceinline__ void xform(const Cam &c, const double *__restrict__ v, double out[3]) {
  const double x = __ldg(v), y = __ldg(v + 1), z = __ldg(v + 2);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    out[r] = __dadd_rn(__fma_rn(z, c.R[3 * r + 2], __fma_rn(y, c.R[3 * r + 1], __dmul_rn(x, c.R[3 * r]))),
                       c.T[r]);
}

__device__ __forceinline__ void tri_cam(const tfb_scene &sc, const Cam &cam, int64_t t, double P[3][3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int64_t vi = __ldg(sc.triangles + 3 * t + k);
    xform(cam, sc.vertices + 3 * vi, P[k]);
  }
}

// rasterizer.py:62-82 (Sutherland–Hodgman against z >= NEAR_PLANE).
__device__ int clip_near(const double P[3][3], double op[4][3], double ob[4][3]) {
  int n = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int k1 = (k + 1) % 3;
    const double *a = P[k], *b = P[k1];
    const bool ina = a[2] >= kNearPlane, inb = b[2] >= kNearPlane;
    if (ina) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        op[n][q] = a[q];
        ob[n][q] = (q == k) ? 1.0 : 0.0;
      }
      ++n;
    }
    if (ina != inb) {
      const double tt = __ddiv_rn(__dsub_rn(kNearPlane, a[2]), __dsub_rn(b[2], a[2]));
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        op[n][q] = __dadd_rn(a[q], __dmul_rn(tt, __dsub_rn(b[q], a[q])));
        const double ba = (q == k) ? 1.0 : 0.0, bb = (q == k1) ? 1.0 : 0.0;
        ob[n][q] = __dadd_rn(ba, __dmul_rn(tt, __dsub_rn(bb, ba)));
      }
      ++n;
    }
  }
  return n;
}

__device__ __forceinline__ bool boundary_accept(double ax, double ay, double bx, double by) {
  // rasterizer.py:85-90
  const double dy = __dsub_rn(by, ay), dx = __dsub_rn(bx, ax);
  return dy > 0.0 || (dy == 0.0 && dx < 0.0);
}

// rasterizer.py:136-164 up to the per-pixel loop.  Returns false when the
// reference would return early (empty bbox, zero or non-finite area).
__device__ bool build_record(const Cam &cam, int W, int H, const double P[3][3], int32_t off, bool clipped, int sub,
                             uint32_t tflags, RecGeom &g, RecMeta &mt) {
  double xs0[3], ys0[3], zs0[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    zs0[k] = P[k][2];
    xs0[k] = __dadd_rn(__dmul_rn(__ddiv_rn(P[k][0], zs0[k]), cam.fx), cam.cx);  // :138
    ys0[k] = __dadd_rn(__dmul_rn(__ddiv_rn(P[k][1], zs0[k]), cam.fy), cam.cy);  // :139
  }
  const double xmin = fmin(fmin(xs0[0], xs0[1]), xs0[2]), xmax = fmax(fmax(xs0[0], xs0[1]), xs0[2]);
  const double ymin = fmin(fmin(ys0[0], ys0[1]), ys0[2]), ymax = fmax(fmax(ys0[0], ys0[1]), ys0[2]);
  const double x0d = fmax(ceil(__dsub_rn(xmin, 0.5)), 0.0);
  const double x1d = fmin(floor(__dsub_rn(xmax, 0.5)), (double)(W - 1));
  const double y0d = fmax(ceil(__dsub_rn(ymin, 0.5)), 0.0);
  const double y1d = fmin(floor(__dsub_rn(ymax, 0.5)), (double)(H - 1));
  if (!(x0d <= x1d) || !(y0d <= y1d)) return false;  // :145
  double area2 = __dsub_rn(__dmul_rn(__dsub_rn(xs0[1], xs0[0]), __dsub_rn(ys0[2], ys0[0])),
                           __dmul_rn(__dsub_rn(ys0[1], ys0[0]), __dsub_rn(xs0[2], xs0[0])));  // :148
  if (area2 == 0.0 || !isfinite(area2)) return false;                                           // :149
  const bool re = !(area2 > 0.0);                                                             // :151
  const int o1 = re ? 2 : 1, o2 = re ? 1 : 2;
  g.xs[0] = xs0[0]; g.xs[1] = xs0[o1]; g.xs[2] = xs0[o2];
  g.ys[0] = ys0[0]; g.ys[1] = ys0[o1]; g.ys[2] = ys0[o2];
  g.zs[0] = zs0[0]; g.zs[1] = zs0[o1]; g.zs[2] = zs0[o2];
  g.area2 = fabs(area2);
  uint32_t flags = tflags | (re ? 8u : 0u) | (clipped ? 16u : 0u) | ((uint32_t)sub << 7);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    g.dX[k] = __dsub_rn(g.xs[b], g.xs[a]);
    g.dY[k] = __dsub_rn(g.ys[b], g.ys[a]);
    if (boundary_accept(g.xs[a], g.ys[a], g.xs[b], g.ys[b])) flags |= 1u << k;
  }
  mt.x0 = (int16_t)x0d;
  mt.x1 = (int16_t)x1d;
  mt.y0 = (int16_t)y0d;
  mt.y1 = (int16_t)y1d;
  mt.off = off;
  mt.flags = flags;
  return true;
}

// A stored record whose tile-bin appends are still to be issued.  k_setup
// batches the appends of several records so their returning atomics are in
// flight together instead of one dependent round trip per record.
struct Pend {
  uint32_t slot;  // record index (records of a frame are allocated densely)
  uint32_t tx, ty;  // first tile (x | last x << 16), (y | last y << 16)
  bool valid;
};

__device__ __forceinline__ void store_record(const Work &w, int f, uint32_t slot, uint32_t key, const RecGeom &g,
                                             const RecMeta &mt, Pend &pd) {
  RecStore *dst = w.rec + (int64_t)f * w.rs + slot;
  dst->meta = mt;
  dst->key = key;
  double2 *d2 = reinterpret_cast<double2 *>(dst->xs);
  const double *gd = reinterpret_cast<const double *>(&g);  // xs, ys, zs lead RecGeom
#pragma unroll
  for (int q = 0; q < 4; ++q) d2[q] = make_double2(gd[2 * q], gd[2 * q + 1]);
  dst->zs[2] = g.zs[2];
  pd.slot = slot;
  pd.tx = (uint32_t)(mt.x0 / kTW) | ((uint32_t)(mt.x1 / kTW) << 16);
  pd.ty = (uint32_t)(mt.y0 / kTH) | ((uint32_t)(mt.y1 / kTH) << 16);
  pd.valid = true;
}

// an allocated slot whose (sub)triangle produced no record (empty bbox, zero
// area, or the second fan slot of a 3-vertex clip): empty bbox, never binned
__device__ __forceinline__ void store_hole(const Work &w, int f, uint32_t slot) {
  RecStore *dst = w.rec + (int64_t)f * w.rs + slot;
  RecMeta e;
  e.x0 = 1;
  e.x1 = 0;
  e.y0 = 1;
  e.y1 = 0;
  e.off = 0;
  e.flags = 0;
  dst->meta = e;
  dst->key = kNoKey;
}

__device__ __forceinline__ void bin_put(const Work &w, int f, int ntiles, int tile, uint32_t pos, uint32_t slot) {
  if (pos < (uint64_t)w.bincap) w.list[((int64_t)f * ntiles + tile) * w.bincap + pos] = slot;
}

// Per (frame, vertex): a clip outcode of the camera-space position (FMA order
// of geometry.py:161).  bit 0: z < NEAR_PLANE; bits 1-4: the vertex projects
// more than 1/4 pixel beyond the left / right / top / bottom image edge (set
// only when z >= NEAR_PLANE, tested without divisions).  A triangle whose
// three outcodes share bit 0 is skipped exactly as rasterizer.py:111 skips it;
// one sharing an edge bit has an empty bbox in the reference
// (rasterizer.py:141-146) — the 1/4 px margin dwarfs the rounding of these
// products, so no visible triangle is dropped.
__device__ __forceinline__ uint32_t vertex_code(const Cam &cam, const double P[3], int W, int H) {
  if (P[2] < kNearPlane) return 1u;
  const double z = P[2];
  return ((P[0] * cam.fx + (cam.cx - 0.25) * z < 0.0) ? 2u : 0u) |
         ((P[0] * cam.fx + (cam.cx - ((double)W - 0.25)) * z > 0.0) ? 4u : 0u) |
         ((P[1] * cam.fy + (cam.cy - 0.25) * z < 0.0) ? 8u : 0u) |
         ((P[1] * cam.fy + (cam.cy - ((double)H - 0.25)) * z > 0.0) ? 16u : 0u);
}

// Record(s) of one surviving triangle t with camera-space vertices P (rasterizer.py:113-164):
// one record at `slot` when no vertex is behind the near plane, else the clip fan's two
// halves at slot and slot + 1 (holes where a half produces nothing).  p0 / p1 receive the
// records' pending tile-bin appends.
__device__ __forceinline__ void setup_candidate(const tfb_scene &sc, const Cam &cam, int W, int H, const Work &w, int f,
                                                int64_t t, const double P[3][3], bool unclipped, uint32_t slot,
                                                Pend &p0, Pend &p1) {
  RecGeom g;
  RecMeta mt;
  const uint32_t tflags = ((uint32_t)__ldg(sc.origins + t) << 5) | ((uint32_t)__ldg(sc.steps + t) << 16);
  const int32_t toff = (int32_t)__ldg(sc.offsets + t);
  if (unclipped) {
    if (build_record(cam, W, H, P, toff, false, 0, tflags, g, mt)) store_record(w, f, slot, (uint32_t)(2 * t), g, mt, p0);
    else store_hole(w, f, slot);
  } else {
    double op[4][3], ob[4][3];
    const int n = clip_near(P, op, ob);
    for (int k = 1; k <= 2; ++k) {  // fan (0, k, k+1), rasterizer.py:119-122
      bool ok = false;
      if (k + 1 < n) {
        double S[3][3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          S[0][q] = op[0][q];
          S[1][q] = op[k][q];
          S[2][q] = op[k + 1][q];
        }
        ok = build_record(cam, W, H, S, toff, true, k - 1, tflags, g, mt);
      }
      if (ok) store_record(w, f, slot + (k - 1), (uint32_t)(2 * t + (k - 1)), g, mt, k == 1 ? p0 : p1);
      else store_hole(w, f, slot + (k - 1));
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_verts(tfb_scene sc, const double *__restrict__ cams, int W, int H,
                                                    Work w) {
  const int f = blockIdx.y;
  __shared__ Cam cam;
  load_cam(cam, cams, f);
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (v >= sc.num_vertices) return;
  double P[3];
  xform(cam, sc.vertices + 3 * v, P);
  w.vcode[(int64_t)f * w.nv + v] = (uint8_t)vertex_code(cam, P, W, H);
}

// Per (frame, triangle), light and fully occupied: the AND of the three
// vertex outcodes decides whether the triangle can produce a record at all;
// survivors are appended (one global atomic per block) to the frame's
// candidate list.
constexpr int kCullPer = 4;  // triangles per k_cull thread (independent loads in flight)

__global__ void __launch_bounds__(kThreads) k_cull(tfb_scene sc, Work w) {
  const int f = blockIdx.y;
  __shared__ uint32_t wtot[kThreads / 32];
  __shared__ uint32_t base_a, base_b;
  const int64_t t0 = (int64_t)blockIdx.x * kThreads * kCullPer + threadIdx.x;
  const uint8_t *vc = w.vcode + (int64_t)f * w.nv;
  int32_t vi[kCullPer][3];
#pragma unroll
  for (int k = 0; k < kCullPer; ++k) {
    const int64_t t = t0 + (int64_t)k * kThreads;
#pragma unroll
    for (int q = 0; q < 3; ++q) vi[k][q] = t < sc.num_triangles ? __ldg(sc.triangles + 3 * t + q) : -1;
  }
  unsigned cmask = 0, nmask = 0;  // bit k: triangle t0 + k * kThreads is a candidate / has a vertex behind
#pragma unroll
  for (int k = 0; k < kCullPer; ++k) {
    if (vi[k][0] < 0) continue;
    const uint32_t c0 = vc[vi[k][0]], c1 = vc[vi[k][1]], c2 = vc[vi[k][2]];
    if ((c0 & c1 & c2) == 0u) {  // not all behind the near plane nor beyond one image edge
      cmask |= 1u << k;
      nmask |= ((c0 | c1 | c2) & 1u) << k;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // unclipped survivors counted in the low half, near-clipped ones in the high half
  const uint32_t mine = (uint32_t)__popc(cmask & ~nmask) | ((uint32_t)__popc(cmask & nmask) << 16);
  uint32_t incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int i = 0; i < kThreads / 32; ++i) {
      const uint32_t v = wtot[i];
      wtot[i] = s;
      s += v;
    }
    base_a = (s & 0xffffu) ? atomicAdd(w.fcnt + 4 * f + 2, s & 0xffffu) : 0u;
    base_b = (s >> 16) ? atomicAdd(w.fcnt + 4 * f + 3, s >> 16) : 0u;
  }
  __syncthreads();
  // entries carry the vertex ids and the near-clip flag, so k_setup needs no
  // further dependent loads before its transform
  const uint32_t ex = wtot[warp] + incl - mine;
  uint4 *const list = w.cand + (int64_t)f * (w.rs / 2);
  uint32_t ia = base_a + (ex & 0xffffu);                       // front, ascending
  int64_t ib = w.rs / 2 - 1 - (int64_t)(base_b + (ex >> 16));  // back, descending
#pragma unroll
  for (int k = 0; k < kCullPer; ++k)
    if ((cmask >> k) & 1u) {
      const bool nc = (nmask >> k) & 1u;
      const uint4 e = make_uint4((uint32_t)(t0 + (int64_t)k * kThreads) | ((uint32_t)nc << 31), (uint32_t)vi[k][0],
                                 (uint32_t)vi[k][1], (uint32_t)vi[k][2]);
      if (nc) list[ib--] = e;
      else list[ia++] = e;
    }
}

// ---- Cluster cull (scenes with tfb_scene clusters; replaces k_verts + k_cull) ----
//
// k_ccull, per (frame, cluster): the camera transform of the 8 corners of the
// cluster's world AABB.  Each outcode condition of k_verts is a half-space in
// camera space (z < NEAR_PLANE, or beyond an image edge by 1/4 px as the plane
// through the camera centre), and camera coordinates are affine in world
// coordinates, so when all 8 corners lie in one such half-space every vertex of
// every triangle of the cluster does.  Then every triangle is either skipped by
// rasterizer.py:111 or, clipped or not, has all of its (clipped) polygon
// projecting beyond the edge, i.e. an empty bbox (rasterizer.py:141-146) -- it
// produces nothing, as in the reference.  The corner tests carry a slack of
// 1e-12 of the magnitudes involved, far above the rounding of the corner and
// vertex transforms, so only clusters that are strictly outside are culled.
constexpr int kCluster = 64;  // triangle slots per cluster

__device__ __forceinline__ void xform_point(const Cam &c, const double p[3], double out[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    out[r] = __dadd_rn(__fma_rn(p[2], c.R[3 * r + 2], __fma_rn(p[1], c.R[3 * r + 1], __dmul_rn(p[0], c.R[3 * r]))),
                       c.T[r]);
}

__global__ void __launch_bounds__(kThreads) k_ccull(tfb_scene sc, const double *__restrict__ cams, int W, int H,
                                                    Work w) {
  const int f = blockIdx.y;
  __shared__ Cam cam;
  load_cam(cam, cams, f);
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  bool keep = false;
  if (c < sc.num_clusters) {
    static_assert(sizeof(tfb_cluster) == 1856, "tfb_cluster layout");
    const double *bx = sc.clusters[c].box;
    const double lo[3] = {__ldg(bx), __ldg(bx + 1), __ldg(bx + 2)};
    const double hi[3] = {__ldg(bx + 3), __ldg(bx + 4), __ldg(bx + 5)};
    double rmax = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) rmax = fmax(rmax, fabs(cam.R[i]));
    const double tmag = fabs(cam.T[0]) + fabs(cam.T[1]) + fabs(cam.T[2]);
    const double kx = fabs(cam.fx) + fabs(cam.cx) + (double)W + 1.0, ky = fabs(cam.fy) + fabs(cam.cy) + (double)H + 1.0;
    uint32_t all = 31u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double p[3] = {(i & 1) ? hi[0] : lo[0], (i & 2) ? hi[1] : lo[1], (i & 4) ? hi[2] : lo[2]};
      double P[3];
      xform_point(cam, p, P);
      const double z = P[2];
      const double tol = 1e-12 * ((fabs(p[0]) + fabs(p[1]) + fabs(p[2])) * rmax + tmag) + 1e-300;
      const double sx = kx * tol + 1e-12 * (fabs(P[0] * cam.fx) + (fabs(cam.cx) + (double)W) * fabs(z));
      const double sy = ky * tol + 1e-12 * (fabs(P[1] * cam.fy) + (fabs(cam.cy) + (double)H) * fabs(z));
      uint32_t m = (z < kNearPlane - tol) ? 1u : 0u;
      m |= (P[0] * cam.fx + (cam.cx - 0.25) * z < -sx) ? 2u : 0u;
      m |= (P[0] * cam.fx + (cam.cx - ((double)W - 0.25)) * z > sx) ? 4u : 0u;
      m |= (P[1] * cam.fy + (cam.cy - 0.25) * z < -sy) ? 8u : 0u;
      m |= (P[1] * cam.fy + (cam.cy - ((double)H - 0.25)) * z > sy) ? 16u : 0u;
      all &= m;
    }
    keep = all == 0u;  // (a NaN corner sets no bit: kept)
  }
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(bal) - 1) base = atomicAdd(w.fcnt + 4 * f, (uint32_t)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
  if (keep) w.csurv[(int64_t)f * w.ncl + base + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)c;
}

// k_ccands, per (frame, surviving cluster): the outcodes of the cluster's
// distinct vertices (the same transform and conditions as k_verts) into shared
// memory, then per triangle slot the test of k_cull, survivors appended the
// same way (one pair of atomics per warp).  Blocks take four clusters at a
// time and stride over the frame's survivors.
constexpr int kCV = 128;  // vertex slots per cluster (tfb_cluster::verts)

#ifndef TFB_CCANDS_MINB
#define TFB_CCANDS_MINB 8  // 32 registers: 8 blocks (64 warps) per SM hide the cluster -> vertex -> append chain
#endif
__global__ void __launch_bounds__(kThreads, TFB_CCANDS_MINB) k_ccands(tfb_scene sc, const double *__restrict__ cams, int W, int H,
                                                     Work w) {
  const int f = blockIdx.y;
  constexpr int kPer = kThreads / kCluster;
  __shared__ Cam cam;
  __shared__ uint8_t scode[kPer][kCV];
  load_cam(cam, cams, f);
  __syncthreads();
  const uint32_t nsurv = w.fcnt[4 * f];
  const uint32_t *cs = w.csurv + (int64_t)f * w.ncl;
  uint4 *const list = w.cand + (int64_t)f * (w.rs / 2);
  const int lane = threadIdx.x & 31, sub = threadIdx.x / kCluster, slot = threadIdx.x % kCluster;
  for (uint32_t g0 = blockIdx.x * kPer; g0 < nsurv; g0 += gridDim.x * kPer) {
    const uint32_t gi = g0 + sub;
    const tfb_cluster *cl = gi < nsurv ? sc.clusters + __ldg(cs + gi) : nullptr;
    int4 tr = make_int4(-1, 0, 0, 0);
    uint32_t loc = 0;
    if (cl) {
      tr = __ldg(reinterpret_cast<const int4 *>(cl->tri[slot]));
      loc = __ldg(cl->local + slot);
      // the vertex ids are read unconditionally (all 128 slots exist), in flight
      // with the count; only the first nverts are transformed
      int32_t vid[kCV / kCluster];
#pragma unroll
      for (int k = 0; k < kCV / kCluster; ++k) vid[k] = __ldg(cl->verts + slot + k * kCluster);
      const int nv = __ldg(&cl->nverts);
#pragma unroll
      for (int k = 0; k < kCV / kCluster; ++k) {
        const int j = slot + k * kCluster;
        if (j < nv) {
          double P[3];
          xform(cam, sc.vertices + 3 * (int64_t)vid[k], P);
          scode[sub][j] = (uint8_t)vertex_code(cam, P, W, H);
        }
      }
    }
    __syncthreads();
    bool cand = false, nc = false;
    if (tr.x >= 0) {
      const uint32_t c0 = scode[sub][loc & 0xffu], c1 = scode[sub][(loc >> 8) & 0xffu],
                     c2 = scode[sub][(loc >> 16) & 0xffu];
      cand = (c0 & c1 & c2) == 0u;
      nc = ((c0 | c1 | c2) & 1u) != 0u;
    }
    const unsigned ba = __ballot_sync(0xffffffffu, cand && !nc), bb = __ballot_sync(0xffffffffu, cand && nc);
    uint32_t pa = 0, pb = 0;
    if (lane == 0) {
      if (ba) pa = atomicAdd(w.fcnt + 4 * f + 2, (uint32_t)__popc(ba));
      if (bb) pb = atomicAdd(w.fcnt + 4 * f + 3, (uint32_t)__popc(bb));
    }
    pa = __shfl_sync(0xffffffffu, pa, 0);
    pb = __shfl_sync(0xffffffffu, pb, 0);
    if (cand) {
      const unsigned below = (1u << lane) - 1u;
      const uint4 e = make_uint4((uint32_t)tr.x | ((nc ? 1u : 0u) << 31), (uint32_t)tr.y, (uint32_t)tr.z,
                                 (uint32_t)tr.w);
      if (nc) list[w.rs / 2 - 1 - (int64_t)(pb + __popc(bb & below))] = e;
      else list[pa + __popc(ba & below)] = e;
    }
    __syncthreads();  // scode reused by the next group
  }
}

// Per surviving (frame, triangle): near clip + fan, projection, bbox, signed
// area, CCW reorder and edge setup (rasterizer.py:113-164) into 96-byte
// records (see Work::rec for the slots); tile bins filled.
#ifndef TFB_SETUP_PER
#define TFB_SETUP_PER 2
#endif
constexpr int kSetupPer = TFB_SETUP_PER;  // candidates per k_setup thread (their bin appends are batched)
#ifndef TFB_SETUP_FLAT
#define TFB_SETUP_FLAT 1
#endif
#ifndef TFB_SETUP_WIDE
#define TFB_SETUP_WIDE 8
#endif
constexpr int kSetupWide = TFB_SETUP_WIDE;  // records over more tiles are binned by the whole warp
// the flat deal packs each record's further-tile count into 16-bit halves of two words
static_assert(!TFB_SETUP_FLAT || kSetupPer == 2, "TFB_SETUP_FLAT packs exactly two records per thread");

__global__ void __launch_bounds__(kThreads, TFB_SETUP_MINB) k_setup(tfb_scene sc, const double *__restrict__ cams, int W,
                                                    int H, int TX, int ntiles, Work w) {
  const int f = blockIdx.y;
  __shared__ Cam cam;
  const uint32_t na = w.fcnt[4 * f + 2], ncand = na + w.fcnt[4 * f + 3];
  // the grid is sized for a generous survivor fraction: blocks past the frame's
  // survivors leave before staging the camera
  if ((uint64_t)blockIdx.x * kThreads * kSetupPer >= ncand) return;
  load_cam(cam, cams, f);
  __syncthreads();
  const int64_t mc = w.rs / 2;  // survivor list length (m)
  const uint4 *cl = w.cand + (int64_t)f * mc;
  // candidate prologue: triangle, vertex ids, outcodes -> 1 record slot if no vertex is
  // behind the near plane, else 2 (the fan of rasterizer.py:119-122 has at most two)
  struct Cand {
    int64_t t, i0, i1, i2;
    uint32_t nslot, slot;
    bool unclipped;
  };
  // survivor i: the i-th unclipped one (cand index i, record slot i) or, past them, a
  // near-clipped one from the back (cand index c, record slots 2c and 2c + 1)
  auto head = [&](uint32_t i, Cand &c) {
    c.nslot = 0;
    if (i >= ncand) return;
    const int64_t ci = i < na ? (int64_t)i : mc - 1 - (int64_t)(i - na);
    c.slot = i < na ? (uint32_t)ci : (uint32_t)(2 * ci);
    const uint4 e = cl[ci];
    c.t = e.x & 0x7fffffffu;
    c.i0 = e.y;
    c.i1 = e.z;
    c.i2 = e.w;
    c.unclipped = (e.x >> 31) == 0u;  // zmin >= NEAR_PLANE (k_cull's outcode bit 0)
    c.nslot = c.unclipped ? 1u : 2u;
  };
  auto one = [&](const Cand &c, Pend &p0, Pend &p1) {
    p0.valid = p1.valid = false;
    if (!c.nslot) return;
    // camera-space vertices recomputed here (bit-identical to k_verts' transform): the
    // vertex array is L2-resident across frames, a per-frame camera-space copy is not
    double P[3][3];
    xform(cam, sc.vertices + 3 * c.i0, P[0]);
    xform(cam, sc.vertices + 3 * c.i1, P[1]);
    xform(cam, sc.vertices + 3 * c.i2, P[2]);
    setup_candidate(sc, cam, W, H, w, f, c.t, P, c.unclipped, c.slot, p0, p1);
  };
  uint32_t *tc = w.tile_count + (int64_t)f * ntiles;
  const uint32_t stride = gridDim.x * kThreads * kSetupPer;
  for (uint32_t c0 = blockIdx.x * kThreads * kSetupPer + threadIdx.x; c0 < ncand; c0 += stride) {
    const unsigned act = __activemask();
    const int lane = threadIdx.x & 31;
    Cand cd[kSetupPer];
#pragma unroll
    for (int k = 0; k < kSetupPer; ++k) head(c0 + k * kThreads, cd[k]);
    // record slots follow from the survivor lists' layout: no allocation round trip
    Pend p[2 * kSetupPer];
#pragma unroll
    for (int k = 0; k < kSetupPer; ++k) one(cd[k], p[2 * k], p[2 * k + 1]);
    // first-tile appends of all pending records in flight together (one atomic per
    // distinct tile per warp: neighbouring candidates mostly share a tile), then the rest
    uint32_t pos[2 * kSetupPer];
    unsigned peers[2 * kSetupPer];
#pragma unroll
    for (int e = 0; e < 2 * kSetupPer; ++e) {
      const int tile = p[e].valid ? (int)(p[e].ty & 0xffffu) * TX + (int)(p[e].tx & 0xffffu) : -1 - lane;
      peers[e] = __match_any_sync(act, tile);
      pos[e] = 0u;
      if (p[e].valid && lane == __ffs(peers[e]) - 1) pos[e] = atomicAdd(tc + tile, (uint32_t)__popc(peers[e]));
    }
#pragma unroll
    for (int e = 0; e < 2 * kSetupPer; ++e)
      pos[e] = __shfl_sync(act, pos[e], __ffs(peers[e]) - 1) + __popc(peers[e] & ((1u << lane) - 1u));
#if TFB_SETUP_FLAT
    if (act == 0xffffffffu) {
      // Full warp: the (record, further tile) pairs of all its pending records are
      // numbered warp-wide and dealt round-robin to the lanes, so every lane has
      // at most ceil(pairs / 32) append round trips in flight one after another
      // instead of a thread walking its own records' tiles serially.
      uint32_t ext = 0, ext01 = 0, ext23 = 0;  // further tiles per record (16-bit packed)
#pragma unroll
      for (int e = 0; e < 2 * kSetupPer; ++e) {
        uint32_t n = 0;
        if (p[e].valid) {
          const uint32_t nx = (p[e].tx >> 16) - (p[e].tx & 0xffffu) + 1u, ny = (p[e].ty >> 16) - (p[e].ty & 0xffffu) + 1u;
          n = nx * ny - 1u;
          bin_put(w, f, ntiles, (int)(p[e].ty & 0xffffu) * TX + (int)(p[e].tx & 0xffffu), pos[e], p[e].slot);
        }
        n = min(n, 0xffffu);  // records over > 65535 tiles: the rest below
        if (e < 2) ext01 |= n << (16 * e);
        else ext23 |= n << (16 * (e - 2));
        ext += n;
      }
      uint32_t incl = ext;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t q0 = 0; q0 < total; q0 += 32) {
        const uint32_t q = q0 + lane;
        // owner: the first lane whose inclusive prefix exceeds q
        int lo = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
          if (v <= q) lo += step;
        }
        const uint32_t o_incl = __shfl_sync(0xffffffffu, incl, lo), o_ext = __shfl_sync(0xffffffffu, ext, lo);
        const uint32_t o01 = __shfl_sync(0xffffffffu, ext01, lo), o23 = __shfl_sync(0xffffffffu, ext23, lo);
        uint32_t rtx[2 * kSetupPer], rty[2 * kSetupPer], rslot[2 * kSetupPer];
#pragma unroll
        for (int e = 0; e < 2 * kSetupPer; ++e) {
          rtx[e] = __shfl_sync(0xffffffffu, p[e].tx, lo);
          rty[e] = __shfl_sync(0xffffffffu, p[e].ty, lo);
          rslot[e] = __shfl_sync(0xffffffffu, p[e].slot, lo);
        }
        if (q < total) {
          uint32_t r = q - (o_incl - o_ext);  // index among the owner's further tiles
          uint32_t tx = 0, ty = 0, slot = 0, k = 0;
          bool found = false;
#pragma unroll
          for (int e = 0; e < 2 * kSetupPer; ++e) {
            const uint32_t n = ((e < 2 ? o01 : o23) >> (16 * (e & 1))) & 0xffffu;
            if (!found && r < n) {
              tx = rtx[e];
              ty = rty[e];
              slot = rslot[e];
              k = r + 1u;  // tile k of the record's box (0 = the first, appended above)
              found = true;
            } else if (!found) {
              r -= n;
            }
          }
          const uint32_t x0 = tx & 0xffffu, nx = (tx >> 16) - x0 + 1u, y0 = ty & 0xffffu;
          const int tile = (int)((y0 + k / nx) * (uint32_t)TX + x0 + k % nx);
          bin_put(w, f, ntiles, tile, atomicAdd(tc + tile, 1u), slot);
        }
      }
      // a record over more than 65536 tiles (only with absurd image sizes) keeps its own loop
#pragma unroll
      for (int e = 0; e < 2 * kSetupPer; ++e) {
        if (!p[e].valid) continue;
        const int x0 = (int)(p[e].tx & 0xffffu), nx = (int)(p[e].tx >> 16) - x0 + 1;
        const int y0 = (int)(p[e].ty & 0xffffu), ny = (int)(p[e].ty >> 16) - y0 + 1;
        for (int i = 0x10000; i < nx * ny; ++i) {
          const int tile = (y0 + i / nx) * TX + x0 + i % nx;
          bin_put(w, f, ntiles, tile, atomicAdd(tc + tile, 1u), p[e].slot);
        }
      }
      continue;
    }
#endif
    // the other tiles: a thread appends its own small records (a few round trips);
    // a record over more than kSetupWide tiles is appended by the whole warp, one
    // atomic per lane in flight at a time (a large triangle spans tens of tiles)
    unsigned wide = 0u;  // bit e: record e goes to the warp
#pragma unroll
    for (int e = 0; e < 2 * kSetupPer; ++e) {
      if (!p[e].valid) continue;
      const int x0 = (int)(p[e].tx & 0xffffu), x1 = (int)(p[e].tx >> 16);
      const int y0 = (int)(p[e].ty & 0xffffu), y1 = (int)(p[e].ty >> 16);
      bin_put(w, f, ntiles, y0 * TX + x0, pos[e], p[e].slot);
      if ((x1 - x0 + 1) * (y1 - y0 + 1) > kSetupWide) {
        wide |= 1u << e;
        continue;
      }
      for (int ty = y0; ty <= y1; ++ty)
        for (int tx = (ty == y0 ? x0 + 1 : x0); tx <= x1; ++tx) {
          const int tile = ty * TX + tx;
          bin_put(w, f, ntiles, tile, atomicAdd(tc + tile, 1u), p[e].slot);
        }
    }
    for (unsigned todo = __ballot_sync(act, wide != 0u); todo; todo = __ballot_sync(act, wide != 0u)) {
      const int src = __ffs(todo) - 1;
      const int e = __shfl_sync(act, wide ? __ffs(wide) - 1 : 0, src);
      uint32_t mtx = 0, mty = 0, mslot = 0;
#pragma unroll
      for (int k = 0; k < 2 * kSetupPer; ++k)
        if (k == e) {
          mtx = p[k].tx;
          mty = p[k].ty;
          mslot = p[k].slot;
        }
      const uint32_t btx = __shfl_sync(act, mtx, src), bty = __shfl_sync(act, mty, src);
      const uint32_t bslot = __shfl_sync(act, mslot, src);
      if (lane == src) wide &= wide - 1u;
      const int x0 = (int)(btx & 0xffffu), nx = (int)(btx >> 16) - x0 + 1;
      const int y0 = (int)(bty & 0xffffu), ny = (int)(bty >> 16) - y0 + 1;
      // the active lanes (all 32 but in a frame's last, partial warp) split the tiles;
      // tile 0 is the first tile, appended above
      const int rank = __popc(act & ((1u << lane) - 1u)), nact = __popc(act);
      for (int i = 1 + rank; i < nx * ny; i += nact) {
        const int tile = (y0 + i / nx) * TX + x0 + i % nx;
        bin_put(w, f, ntiles, tile, atomicAdd(tc + tile, 1u), bslot);
      }
    }
  }
}

// Tile-bin appends of NP pending records per lane of a (possibly partial) warp: the
// first-tile appends of all of them warp-aggregated (one atomic per distinct tile) and in
// flight together, then each lane appends its small records' further tiles and the whole
// warp those of records spanning more than kSetupWide tiles (k_setup's non-flat path).
template <int NP>
__device__ __forceinline__ void bin_pending(const Work &w, int f, int ntiles, int TX, uint32_t *tc, const Pend (&p)[NP],
                                            unsigned act, int lane) {
  uint32_t pos[NP];
  unsigned peers[NP];
#pragma unroll
  for (int e = 0; e < NP; ++e) {
    const int tile = p[e].valid ? (int)(p[e].ty & 0xffffu) * TX + (int)(p[e].tx & 0xffffu) : -1 - lane;
    peers[e] = __match_any_sync(act, tile);
    pos[e] = 0u;
    if (p[e].valid && lane == __ffs(peers[e]) - 1) pos[e] = atomicAdd(tc + tile, (uint32_t)__popc(peers[e]));
  }
#pragma unroll
  for (int e = 0; e < NP; ++e)
    pos[e] = __shfl_sync(act, pos[e], __ffs(peers[e]) - 1) + __popc(peers[e] & ((1u << lane) - 1u));
  unsigned wide = 0u;  // bit e: record e goes to the warp
#pragma unroll
  for (int e = 0; e < NP; ++e) {
    if (!p[e].valid) continue;
    const int x0 = (int)(p[e].tx & 0xffffu), x1 = (int)(p[e].tx >> 16);
    const int y0 = (int)(p[e].ty & 0xffffu), y1 = (int)(p[e].ty >> 16);
    bin_put(w, f, ntiles, y0 * TX + x0, pos[e], p[e].slot);
    if ((x1 - x0 + 1) * (y1 - y0 + 1) > kSetupWide) {
      wide |= 1u << e;
      continue;
    }
    for (int ty = y0; ty <= y1; ++ty)
      for (int tx = (ty == y0 ? x0 + 1 : x0); tx <= x1; ++tx) {
        const int tile = ty * TX + tx;
        bin_put(w, f, ntiles, tile, atomicAdd(tc + tile, 1u), p[e].slot);
      }
  }
  for (unsigned todo = __ballot_sync(act, wide != 0u); todo; todo = __ballot_sync(act, wide != 0u)) {
    const int src = __ffs(todo) - 1;
    const int e = __shfl_sync(act, wide ? __ffs(wide) - 1 : 0, src);
    uint32_t mtx = 0, mty = 0, mslot = 0;
#pragma unroll
    for (int k = 0; k < NP; ++k)
      if (k == e) {
        mtx = p[k].tx;
        mty = p[k].ty;
        mslot = p[k].slot;
      }
    const uint32_t btx = __shfl_sync(act, mtx, src), bty = __shfl_sync(act, mty, src);
    const uint32_t bslot = __shfl_sync(act, mslot, src);
    if (lane == src) wide &= wide - 1u;
    const int x0 = (int)(btx & 0xffffu), nx = (int)(btx >> 16) - x0 + 1;
    const int y0 = (int)(bty & 0xffffu), ny = (int)(bty >> 16) - y0 + 1;
    const int rank = __popc(act & ((1u << lane) - 1u)), nact = __popc(act);
    for (int i = 1 + rank; i < nx * ny; i += nact) {
      const int tile = (y0 + i / nx) * TX + x0 + i % nx;
      bin_put(w, f, ntiles, tile, atomicAdd(tc + tile, 1u), bslot);
    }
  }
}

// k_ccsetup = k_ccands + k_setup in one pass (TFB_FUSED_SETUP): per (frame, surviving
// cluster) the cluster's distinct vertices are transformed once into shared memory
// (camera space, bit-identical to xform), the outcode test of k_ccands picks the
// candidates, their record slots come from the same front / back appends, and each
// candidate's thread builds its record(s) from the shared positions and bins them -- no
// survivor list round trip through memory, no second gather and transform of the
// vertices (a cluster's ~55 distinct vertices serve its 64 triangles).
#ifndef TFB_CCSETUP_MINB
#define TFB_CCSETUP_MINB 5  // 48 registers: 5 blocks (40 warps) per SM
#endif
#ifndef TFB_CCSETUP_PER
#define TFB_CCSETUP_PER 2  // clusters per k_ccsetup block (64 threads each; 2 measured 1 % ahead of 4 and 1)
#endif
#ifndef TFB_CCSETUP_GRID_DIV
#define TFB_CCSETUP_GRID_DIV 16  // k_ccsetup grid: one pass of blocks covers 1 / DIV of the clusters (8: raster +1-2 %)
#endif
#ifndef TFB_CCSETUP_EARLY
#define TFB_CCSETUP_EARLY 0
#endif
constexpr int kCcsPer = TFB_CCSETUP_PER;
__global__ void __launch_bounds__(kCcsPer * kCluster, TFB_CCSETUP_MINB * 4 / kCcsPer) k_ccsetup(
    tfb_scene sc, const double *__restrict__ cams, int W, int H, int TX, int ntiles, Work w) {
  const int f = blockIdx.y;
  constexpr int kPer = kCcsPer;
  __shared__ Cam cam;
  __shared__ uint8_t scode[kPer][kCV];
  __shared__ double sP[kPer][3][kCV];  // camera-space positions, component-major
  const uint32_t *cs = w.csurv + (int64_t)f * w.ncl;
  const int lane = threadIdx.x & 31, sub = threadIdx.x / kCluster, slot = threadIdx.x % kCluster;
#if TFB_CCSETUP_EARLY
  // the survivor count (and, EARLY >= 2, this thread's first survivor entry, read
  // speculatively: the list has ncl slots) is read in flight with the camera; blocks
  // past the frame's survivors (the grid is sized for a generous fraction) leave first
  const uint32_t nsurv = w.fcnt[4 * f];
  uint32_t cid = 0;
  if (TFB_CCSETUP_EARLY >= 2 && blockIdx.x * kPer + sub < (uint32_t)w.ncl) cid = __ldg(cs + blockIdx.x * kPer + sub);
  if (blockIdx.x * kPer >= nsurv) return;
  load_cam(cam, cams, f);
  __syncthreads();
#else
  load_cam(cam, cams, f);
  __syncthreads();
  const uint32_t nsurv = w.fcnt[4 * f];
#endif
  uint32_t *tc = w.tile_count + (int64_t)f * ntiles;
  const int64_t mc = w.rs / 2;
  for (uint32_t g0 = blockIdx.x * kPer; g0 < nsurv; g0 += gridDim.x * kPer) {
    const uint32_t gi = g0 + sub;
#if TFB_CCSETUP_EARLY >= 2
    const tfb_cluster *cl = gi < nsurv ? sc.clusters + cid : nullptr;
    {  // the next group's entry, in flight with this group's work
      const uint32_t gn = gi + gridDim.x * kPer;
      cid = gn < nsurv ? __ldg(cs + gn) : 0u;
    }
#else
    const tfb_cluster *cl = gi < nsurv ? sc.clusters + __ldg(cs + gi) : nullptr;
#endif
    int4 tr = make_int4(-1, 0, 0, 0);
    uint32_t loc = 0;
    if (cl) {
      tr = __ldg(reinterpret_cast<const int4 *>(cl->tri[slot]));
      loc = __ldg(cl->local + slot);
      int32_t vid[kCV / kCluster];
#pragma unroll
      for (int k = 0; k < kCV / kCluster; ++k) vid[k] = __ldg(cl->verts + slot + k * kCluster);
      const int nv = __ldg(&cl->nverts);
#pragma unroll
      for (int k = 0; k < kCV / kCluster; ++k) {
        const int j = slot + k * kCluster;
        if (j < nv) {
          double P[3];
          xform(cam, sc.vertices + 3 * (int64_t)vid[k], P);
          scode[sub][j] = (uint8_t)vertex_code(cam, P, W, H);
          sP[sub][0][j] = P[0];
          sP[sub][1][j] = P[1];
          sP[sub][2][j] = P[2];
        }
      }
    }
    __syncthreads();
    bool cand = false, nc = false;
    uint32_t l0 = 0, l1 = 0, l2 = 0;
    if (tr.x >= 0) {
      l0 = loc & 0xffu;
      l1 = (loc >> 8) & 0xffu;
      l2 = (loc >> 16) & 0xffu;
      const uint32_t c0 = scode[sub][l0], c1 = scode[sub][l1], c2 = scode[sub][l2];
      cand = (c0 & c1 & c2) == 0u;
      nc = ((c0 | c1 | c2) & 1u) != 0u;
    }
    const unsigned ba = __ballot_sync(0xffffffffu, cand && !nc), bb = __ballot_sync(0xffffffffu, cand && nc);
    uint32_t pa = 0, pb = 0;
    if (lane == 0) {
      if (ba) pa = atomicAdd(w.fcnt + 4 * f + 2, (uint32_t)__popc(ba));
      if (bb) pb = atomicAdd(w.fcnt + 4 * f + 3, (uint32_t)__popc(bb));
    }
    pa = __shfl_sync(0xffffffffu, pa, 0);
    pb = __shfl_sync(0xffffffffu, pb, 0);
    Pend pd[2];
    pd[0].valid = pd[1].valid = false;
    if (cand) {
      // record slots exactly as k_setup derives them from the survivor lists: the i-th
      // unclipped survivor -> slot i, the near-clipped one at back index ci -> 2ci, 2ci + 1
      const unsigned below = (1u << lane) - 1u;
      const uint32_t rslot = nc ? (uint32_t)(2 * (mc - 1 - (int64_t)(pb + __popc(bb & below))))
                                : pa + __popc(ba & below);
      double P[3][3];
      const uint32_t lk[3] = {l0, l1, l2};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        P[k][0] = sP[sub][0][lk[k]];
        P[k][1] = sP[sub][1][lk[k]];
        P[k][2] = sP[sub][2][lk[k]];
      }
      setup_candidate(sc, cam, W, H, w, f, (int64_t)tr.x, P, !nc, rslot, pd[0], pd[1]);
    }
    bin_pending<2>(w, f, ntiles, TX, tc, pd, 0xffffffffu, lane);
    __syncthreads();  // scode / sP reused by the next group
  }
}

#ifdef TFB_RASTER_STATS
// experiment-only histograms (tools/raster_stats.py): [0,16) records per tile /32,
// [16,32) covering records per pixel, [32,48) pairs per tile /256, [48] big tiles
__device__ unsigned long long g_rstats[64];
#define RSTAT(i) atomicAdd(&g_rstats[(i)], 1ull)
#else
#define RSTAT(i) ((void)0)
#endif

struct Outs {
  int32_t *rows;
  uint32_t *hits;
  int32_t *tri;
  int32_t *texel;
  double *depth;
  double *u;
  double *v;
};

// Record geometry views.  RecGeom is 16 doubles: xs[3] ys[3] zs[3] dX[3] dY[3] area2.
enum { kFXs = 0, kFYs = 3, kFZs = 6, kFDX = 9, kFDY = 12, kFA2 = 15, kFields = 16 };
constexpr int kPC = 8;        // covering slots kept per pixel by the pair phase (more: selection by key)
static_assert(kPC >= 4, "the fold's 4-input network reads four kept slots");

struct AosRec {  // one RecGeom (global memory or AoS shared memory)
  const RecGeom *g;
  __device__ __forceinline__ double f(int k) const { return reinterpret_cast<const double *>(g)[k]; }
};

// Record j of a tile staged field-major (lanes reading different records hit
// different banks).  Only xs, ys, zs and |area2| are staged (kStaged fields);
// the edge deltas are re-derived on read exactly as expand_derived forms them.
constexpr int kStaged = 11;
constexpr int kSA2 = 9;   // staged slot of |area2|
constexpr int kSThr = 10;  // staged slot of the sole-candidate threshold (first_win_threshold)
template <int FS>
struct SoaRecT {
  const double *base;
  int j;
  __device__ __forceinline__ double at(int q) const { return base[q * FS + j]; }
  __device__ __forceinline__ double f(int k) const {
    if (k < kFDX) return at(k);
    if (k == kFA2) return at(kSA2);
    const int kk = (k - kFDX) % 3, o = k < kFDY ? kFXs : kFYs;  // dX (xs) or dY (ys)
    return __dsub_rn(at(o + (kk + 2) % 3), at(o + (kk + 1) % 3));
  }
};

// edge functions at one pixel centre, rasterizer.py:161-162
template <typename R>
__device__ __forceinline__ bool edges_at(const R &g, uint32_t flags, double px, double py, double e[3]) {
  bool inside = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3;
    e[k] = __dsub_rn(__dmul_rn(g.f(kFDX + k), __dsub_rn(py, g.f(kFYs + a))),
                     __dmul_rn(g.f(kFDY + k), __dsub_rn(px, g.f(kFXs + a))));
    inside = inside && (e[k] > 0.0 || (e[k] == 0.0 && ((flags >> k) & 1u)));
  }
  return inside;
}

__device__ __forceinline__ double np_max(double a, double b) { return isnan(a) ? a : (a > b ? a : b); }
__device__ __forceinline__ double np_min(double a, double b) { return isnan(a) ? a : (a < b ? a : b); }

// Sequential-fold step for one covering record (rasterizer.py:170-171): the
// reference's exact `z > 0 && z < depth - 1e-9` in float64.
struct Fold {
  double depth, w0, w1, w2;
  int32_t win;  // record slot (smem index or global key), -1 = none
  __device__ __forceinline__ void init() {
    depth = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    w0 = w1 = w2 = 0.0;
    win = -1;
  }
  template <typename R>
  __device__ __forceinline__ void step(const R &g, uint32_t flags, double px, double py, int32_t id) {
    double e[3];
    edges_at(g, flags, px, py, e);
    step_e(g, e, id);
  }
  template <typename R>
  __device__ __forceinline__ void step_e(const R &g, const double e[3], int32_t id) {
    // rasterizer.py:166-169; divisions via the branch-free fast path (exact_div.cuh)
    const double z0 = g.f(kFZs), z1 = g.f(kFZs + 1), z2 = g.f(kFZs + 2), a2 = g.f(kFA2);
    bool ok = true;
    double a = ddiv_try(e[0], z0, ok), b = ddiv_try(e[1], z1, ok), c = ddiv_try(e[2], z2, ok);
    double z = ddiv_try(a2, __dadd_rn(__dadd_rn(a, b), c), ok);
    if (!ok) {
      a = __ddiv_rn(e[0], z0);
      b = __ddiv_rn(e[1], z1);
      c = __ddiv_rn(e[2], z2);
      z = __ddiv_rn(a2, __dadd_rn(__dadd_rn(a, b), c));
    }
    if (z > 0.0 && z < __dsub_rn(depth, kDepthTie)) {
      depth = z;
      win = id;
      w0 = a;
      w1 = b;
      w2 = c;
    }
  }
  // A pixel's first (here: only) covering record when no depth plane is wanted.
  // Against depth = +inf the test `z > 0 && z < inf - 1e-9` only asks for a
  // finite positive z = area2 / (a + b + c); with a + b + c > area2 * 1e-300 the
  // quotient is below 1e300, so the division is skipped.  Otherwise the exact step.
  template <typename R>
  __device__ __forceinline__ void first_e(const R &g, const double e[3], int32_t id) {
    const double z0 = g.f(kFZs), z1 = g.f(kFZs + 1), z2 = g.f(kFZs + 2), a2 = g.f(kFA2);
    bool ok = true;
    double a = ddiv_try(e[0], z0, ok), b = ddiv_try(e[1], z1, ok), c = ddiv_try(e[2], z2, ok);
    if (!ok) {
      a = __ddiv_rn(e[0], z0);
      b = __ddiv_rn(e[1], z1);
      c = __ddiv_rn(e[2], z2);
    }
    const double sum = __dadd_rn(__dadd_rn(a, b), c);
    // a2 * 1e300 may overflow to +inf: then sum < inf still bounds z = a2 / sum
    // below by a2 / DBL_MAX > 0; a sum of +inf gives z = 0 (no winner)
    if (sum > __dmul_rn(a2, 1e-300) && sum < __dmul_rn(a2, 1e300)) {
      win = id;
      w0 = a;
      w1 = b;
      w2 = c;
    } else {
      step_e(g, e, id);
    }
  }
};

// Division-free form of first_e's acceptance for a covering record (all e_k >= 0):
// with a2, z_k in [1e-100, 1e100] and max e_k <= 1e100, every quotient e_k / z_k is
// at most 1e200, so sum = (a + b) + c < 1e201 is finite and z = a2 / sum > 1e-301;
// with max e_k >= a2 * max z_k * 1e-50 the largest quotient, and so the sum, is at
// least a2 * 1e-50 * (1 - 2^-53), so z < 1e51.  Then z is finite and positive and
// wins against depth = +inf exactly as the divisions would decide.  The products
// stay in the normal range under these bounds.
template <typename R>
__device__ __forceinline__ bool first_wins_without_divisions(const R &g, const double e[3]) {
  const double z0 = g.f(kFZs), z1 = g.f(kFZs + 1), z2 = g.f(kFZs + 2), a2 = g.f(kFA2);
  // every comparison is false for a NaN operand
  const bool zok = z0 >= 1e-100 && z0 <= 1e100 && z1 >= 1e-100 && z1 <= 1e100 && z2 >= 1e-100 && z2 <= 1e100;
  const double zmax = fmax(fmax(z0, z1), z2);
  const double emax = fmax(fmax(e[0], e[1]), e[2]);
  return zok && a2 >= 1e-100 && a2 <= 1e100 && emax <= 1e100 && emax >= __dmul_rn(__dmul_rn(a2, zmax), 1e-50);
}

// first_wins_without_divisions with the record-only part folded into one number per
// record, formed when the record is staged: a2 * max z_k * 1e-50 when steps = 1 and the
// z_k and a2 ranges hold, else NaN (every comparison against it fails).  A covering
// pixel's sole record then wins without divisions iff max e_k <= 1e100 && max e_k >= thr.
//
// With TFB_FAST_LO = 0 the record also requires |x|, |y| <= 1e40 for its projected
// vertices: every edge value at a pixel centre (|px|, |py| < 2^15) is then a difference of
// two products below 2e40 * (1e40 + 2^15), far under 1e100 even after rounding, so the
// max e_k <= 1e100 half of the test holds by construction and is not evaluated per pixel.
__device__ __forceinline__ double first_win_threshold(const double xs[3], const double ys[3], const double zs[3],
                                                      double a2, uint32_t flags) {
  const double z0 = zs[0], z1 = zs[1], z2 = zs[2];
  const bool zok = z0 >= 1e-100 && z0 <= 1e100 && z1 >= 1e-100 && z1 <= 1e100 && z2 >= 1e-100 && z2 <= 1e100;
  const double zmax = fmax(fmax(z0, z1), z2);
  bool ok = (flags >> 16) == 1u && zok && a2 >= 1e-100 && a2 <= 1e100;
  if (!TFB_FAST_LO)
    ok = ok && fabs(xs[0]) <= 1e40 && fabs(xs[1]) <= 1e40 && fabs(xs[2]) <= 1e40 && fabs(ys[0]) <= 1e40 &&
         fabs(ys[1]) <= 1e40 && fabs(ys[2]) <= 1e40;
  return ok ? __dmul_rn(__dmul_rn(a2, zmax), 1e-50) : __longlong_as_double(0x7ff8000000000000LL);
}

// max e_k <= 1e100 && max e_k >= thr for the (non-NaN) edge values of a covering pair,
// evaluated without branches (the first half only with TFB_FAST_LO, see above)
__device__ __forceinline__ bool first_fast(const double e[3], double thr) {
  const bool hi = (e[0] >= thr) | (e[1] >= thr) | (e[2] >= thr);
  if (!TFB_FAST_LO) return hi;
  const bool lo = (e[0] <= 1e100) & (e[1] <= 1e100) & (e[2] <= 1e100);
  return lo & hi;
}

__device__ __forceinline__ void emit_pixel(const tfb_scene &sc, const Outs &o, int f, int64_t pix, int32_t t,
                                           int32_t texel, int32_t row);

// Winner epilogue, rasterizer.py:177-202: perspective-correct barycentrics of
// the original triangle → (u, v) → texel id → global row; optional planes.
// For an unclipped triangle the barycentric rows are a permutation of the
// identity, so (w0*B0k + w1*B1k) + w2*B2k is exactly w_perm(k) (x*1 = x,
// x*0 = 0, x + 0 = x for the finite w's of a covering record) and the
// products are skipped; of the final normalization b /= b.sum() only the two
// components (u, v) read are divided.
__device__ __forceinline__ void write_pixel(const tfb_scene &sc, const Cam &cam, const Outs &o, int f, int W, int H,
                                            int px_i, int py_i, const Fold &fd, uint32_t flags, int32_t t,
                                            int64_t offset) {
  const int64_t pix = (int64_t)f * W * H + (int64_t)(py_i * W + px_i);
  int32_t row = -1, texel = 0;
  if (fd.win >= 0 && (flags >> 16) == 1u && !o.depth) {
    // steps = 1 and no float planes: the texel is 0 whatever the barycentrics
    // (see the sole-candidate path in k_raster)
    row = (int32_t)offset;
  } else if (fd.win >= 0) {
    const double wsum = __dadd_rn(__dadd_rn(fd.w0, fd.w1), fd.w2);
    double b0, b1, b2;
    if (flags & 16u) {  // clipped: barycentric rows of the fan vertices (rasterizer.py:62-82, 119-122)
      const int sub = (flags >> 7) & 1u;
      double P[3][3], op[4][3], ob[4][3];
      tri_cam(sc, cam, t, P);
      clip_near(P, op, ob);
      double B[3][3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        B[0][q] = ob[0][q];
        B[1][q] = sub ? ob[2][q] : ob[1][q];
        B[2][q] = sub ? ob[3][q] : ob[2][q];
      }
      if (flags & 8u) {  // reorder (0, 2, 1), rasterizer.py:151-152
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double tmp = B[1][q];
          B[1][q] = B[2][q];
          B[2][q] = tmp;
        }
      }
      double nb[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        nb[k] = __dadd_rn(__dadd_rn(__dmul_rn(fd.w0, B[0][k]), __dmul_rn(fd.w1, B[1][k])), __dmul_rn(fd.w2, B[2][k]));
      b0 = __ddiv_rn(nb[0], wsum);
      b1 = __ddiv_rn(nb[1], wsum);
      b2 = __ddiv_rn(nb[2], wsum);
    } else {
      // rows = identity reordered by (0, 1, 2) or (0, 2, 1): b_k = w_perm(k) / wsum
      const double n1 = (flags & 8u) ? fd.w2 : fd.w1, n2 = (flags & 8u) ? fd.w1 : fd.w2;
      bool ok = true;
      b0 = ddiv_try(fd.w0, wsum, ok);
      b1 = ddiv_try(n1, wsum, ok);
      b2 = ddiv_try(n2, wsum, ok);
      if (!ok) {
        b0 = __ddiv_rn(fd.w0, wsum);
        b1 = __ddiv_rn(n1, wsum);
        b2 = __ddiv_rn(n2, wsum);
      }
    }
    if (b0 < 0.0) b0 = 0.0;  // np.clip(b, 0, None)
    if (b1 < 0.0) b1 = 0.0;
    if (b2 < 0.0) b2 = 0.0;
    const double bs = __dadd_rn(__dadd_rn(b0, b1), b2);
    const int origin = (flags >> 5) & 3u;
    const int s = (int)(flags >> 16);
    const double bo = origin == 0 ? b0 : (origin == 1 ? b1 : b2);
    const double bv = origin == 0 ? b2 : (origin == 1 ? b0 : b1);
    bool ok = true;
    double qo = ddiv_try(bo, bs, ok), v = ddiv_try(bv, bs, ok);
    if (!ok) {
      qo = __ddiv_rn(bo, bs);
      v = __ddiv_rn(bv, bs);
    }
    double u = __dsub_rn(1.0, qo);
    u = np_min(np_max(u, 0.0), 1.0);
    v = np_min(np_max(v, 0.0), u);
    int i = (int)__dmul_rn((double)s, u);
    if (i > s - 1) i = s - 1;
    int j = (int)__dmul_rn((double)s, v);
    if (j > i) j = i;
    texel = (i * i + i) / 2 + j;
    row = (int32_t)(offset + texel);
    if (o.depth) {
      o.depth[pix] = fd.depth;
      o.u[pix] = u;
      o.v[pix] = v;
    }
  } else if (o.depth) {
    o.depth[pix] = fd.depth;
    o.u[pix] = 0.0;
    o.v[pix] = 0.0;
  }
  emit_pixel(sc, o, f, pix, fd.win >= 0 ? t : -1, texel, row);
}

// Id planes, the fusion row and the per-frame texel hit count of one pixel
// (t = -1: no triangle, texel 0, row -1).
__device__ __forceinline__ void emit_pixel(const tfb_scene &sc, const Outs &o, int f, int64_t pix, int32_t t,
                                           int32_t texel, int32_t row) {
  if (o.tri) {
    o.tri[pix] = t;
    o.texel[pix] = texel;
  }
  o.rows[pix] = row;
  if (o.hits && row >= 0) {
    // warp-aggregated per-frame texel hit count (fusion.py:135-136)
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, row);
    if ((int)(__ffs(peers) - 1) == (int)(threadIdx.x & 31))
      atomicAdd(o.hits + (int64_t)f * sc.total_texels + row, (uint32_t)__popc(peers));
  }
}

// Shared memory of one tile staged by a CTA of NT threads (at most NT records).
template <int NT>
struct TileSmem {
  static constexpr int FS = NT + 1;  // field stride: the fields of lanes on different records on distinct banks
  double g[kStaged * FS];            // staged records, field-major (SoA): g[q * FS + j]
#if TFB_KEEP_PE
  double pe[3][kTP];                 // edge values of a pixel's (single) covering pair
#endif
  uint8_t pc[kPC][kTP];              // per pixel: slots of its first kPC covering pairs (arrival order)
  uint32_t flags[NT];                // RecMeta::flags
  int32_t off[NT];                   // offsets[t] of the record's triangle (n_x < 2^31)
  Cam cam;
  uint32_t key[NT];
  uint32_t box[NT];                  // tile-relative bbox: x0 | y0 << 8 | w << 16 | h << 24
  uint32_t pre[NT];                  // exclusive prefix of bbox areas
  uint32_t pcnt[kTP];
  uint32_t wtot[NT / 32];
};
static_assert(kTP <= 256, "covering slots are stored as bytes");

// One CTA of kTP threads per kTW x kTH tile with at most kTP records (the common case).
//  1. The tile's records are staged in shared memory in list order (all
//     threads cooperate on the 128-byte copies); bbox-in-tile and area per
//     record, exclusive scan of areas.
//  2. Pair-parallel edge tests: every (record, pixel of its bbox in the tile)
//     pair gets its own thread (one binary search per thread-run), so float64
//     lanes are not wasted on pixels outside a small triangle's bbox.  A
//     covering pair bumps the pixel's candidate count (32-bit smem atomic)
//     and the first kPC = 8 covering slots are kept.
//  3. One thread per pixel: up to eight candidates are ordered by key among
//     the kept slots and folded; with more, the pixel repeatedly selects the
//     smallest covering key above the last folded one — the reference's
//     ascending sequential fold (rasterizer.py:108, 170-171) without sorting.
//  Larger or overflowed tiles are handed to k_raster_big.
template <int NT>
__device__ __forceinline__ void raster_tile(const tfb_scene &sc, const double *__restrict__ cams, int W, int H, int TX,
                                            int ntiles, const Work &w, const Outs &o, int f, int tx, int ty,
                                            unsigned char *raster_smem) {
  static_assert(NT % 32 == 0 && NT <= kTP && kTP % NT == 0, "whole warps, whole pixel passes");
  constexpr int FS = TileSmem<NT>::FS;
  using Rec = SoaRecT<FS>;
  const int tile = ty * TX + tx;
  const int tx0 = tx * kTW, ty0 = ty * kTH;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the bin entry this thread would stage is read speculatively, in flight together
  // with the tile's count (entries past the count are stale and ignored)
  const uint32_t *src = w.list + ((int64_t)f * ntiles + tile) * w.bincap;
  const uint32_t key_spec = tid < (int)min(w.bincap, (int64_t)NT) ? src[tid] : 0u;
  const uint32_t n = w.tile_count[(int64_t)f * ntiles + tile];
  if (n > (uint64_t)w.bincap || n > (uint32_t)NT) {
    if (tid == 0) {
      const uint32_t code = (uint32_t)(f * ntiles + tile);
      if (NT < kTP && n <= (uint64_t)w.bincap && n <= (uint32_t)kTP) {
        const int tier = n <= 64u ? 0 : 1;  // the smallest wider CTA that stages them all
        w.tl[tier * w.tlcap + atomicAdd(w.tcnt + tier, 1u)] = code;
      } else {
        w.big[atomicAdd(w.fcnt + 1, 1u)] = code;
      }
      RSTAT(48);
    }
    return;
  }
  if (tid == 0) RSTAT(min(n / 32u, 15u));
  TileSmem<NT> &S = *reinterpret_cast<TileSmem<NT> *>(raster_smem);
  double *sg = S.g;
  uint32_t *sflags = S.flags;
  int32_t *soff = S.off;
  uint32_t *skey = S.key, *sbox = S.box, *spre = S.pre, *pcnt = S.pcnt, *wtot = S.wtot;
  uint8_t(*pc)[kTP] = S.pc;
#if TFB_KEEP_PE
  double(*pe)[kTP] = S.pe;
#endif
  Cam &cam = S.cam;
  load_cam(cam, cams, f);
#pragma unroll
  for (int q = tid; q < kTP; q += NT) pcnt[q] = 0u;
  const RecStore *recs = w.rec + (int64_t)f * w.rs;
  uint32_t area = 0;
  if (tid < n) {
    // one thread per record: its 96 bytes in six 16-byte loads, the derived
    // fields formed in registers, all 16 fields stored field-major
    const double2 *r2 = reinterpret_cast<const double2 *>(recs + key_spec);  // bin entry = record index
    double v[12];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double2 d = __ldg(r2 + q);
      v[2 * q] = d.x;
      v[2 * q + 1] = d.y;
    }
    const RecMeta mt = unpack_meta(v[0], v[1]);
    const uint32_t key = (uint32_t)(unsigned long long)__double_as_longlong(v[11]);  // RecStore::key
    double dX[3], dY[3], a2;
    expand_derived(v + 2, v + 5, dX, dY, a2);
#pragma unroll
    for (int q = 0; q < 9; ++q) sg[q * FS + tid] = v[2 + q];
    sg[kSA2 * FS + tid] = a2;
    sg[kSThr * FS + tid] = first_win_threshold(v + 2, v + 5, v + 8, a2, mt.flags);
    skey[tid] = key;
    sflags[tid] = mt.flags;
    soff[tid] = mt.off;
    const int bx0 = max((int)mt.x0, tx0) - tx0, bx1 = min((int)mt.x1, tx0 + kTW - 1) - tx0;
    const int by0 = max((int)mt.y0, ty0) - ty0, by1 = min((int)mt.y1, ty0 + kTH - 1) - ty0;
    const uint32_t bw = (uint32_t)(bx1 - bx0 + 1), bh = (uint32_t)(by1 - by0 + 1);
    sbox[tid] = (uint32_t)bx0 | ((uint32_t)by0 << 8) | (bw << 16) | (bh << 24);
    area = bw * bh;
  }
  uint32_t total = 0;
  if (n <= 32u) {
    // all records sit in warp 0: it scans their areas alone, one barrier publishes
    if (warp == 0) {
      uint32_t incl = area;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      spre[tid] = incl - area;
      if (lane == 31) wtot[0] = incl;
    }
    __syncthreads();
    total = wtot[0];
  } else {
    uint32_t incl = area;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      const uint32_t v = wtot[i];
      wbase += i < warp ? v : 0u;
      total += v;
    }
    spre[tid] = wbase + incl - area;
    __syncthreads();
  }

  if (tid == 0) RSTAT(32 + min(total / 256u, 15u));
  // pair-parallel edge tests in warp windows: a window is 32 consecutive (record, pixel of
  // its bbox) pairs, lane l taking pair base + l, and each warp walks a contiguous range of
  // windows.  The records starting inside a window come from one shared-memory load per
  // lane and a warp OR-reduction, so a lane finds its record with a popcount (no per-lane
  // search), and all lanes run the same straight-line test (no per-lane row / record
  // refills diverging across the warp).
  {
    const uint32_t nwin = (total + 31u) >> 5;
    const uint32_t wper = (nwin + (NT / 32) - 1) / (NT / 32);
    const uint32_t wbeg = (uint32_t)warp * wper, wend = min(wbeg + wper, nwin);
    if (wbeg < wend) {
      const unsigned upto = (2u << lane) - 1u;
      // jb: the record holding pair base - 1 (areas are >= 1: every binned bbox meets the
      // tile), i.e. the number of records starting at or before it, less one
      int jb = -1;
      if (wbeg > 0u) {
        const uint32_t q = (wbeg << 5) - 1u;
        for (int r0 = 0; r0 < (int)n; r0 += 32)
          jb += __popc(__ballot_sync(0xffffffffu, r0 + lane < (int)n && spre[r0 + lane] <= q));
      }
      for (uint32_t wi = wbeg; wi < wend; ++wi) {
        const uint32_t base = wi << 5;
        const int jc = jb + 1 + lane;
        unsigned bit = 0u;
        if (jc < (int)n) {
          const uint32_t st = spre[jc];
          if (st < base + 32u) bit = 1u << (st - base);
        }
        const unsigned starts = __reduce_or_sync(0xffffffffu, bit);
        const int j = jb + __popc(starts & upto);
        jb += __popc(starts);
        const uint32_t p = base + (uint32_t)lane;
        if (p < total) {
          const uint32_t b = sbox[j];
          const int local = (int)(p - spre[j]);
          const int bw = (int)((b >> 16) & 0xffu);
          // local / bw (local < 2^15, bw <= 255): (local + 0.5) / bw sits >= 0.5 / bw from an
          // integer, far above the error of the approximate reciprocal and the product
          float rbw;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rbw) : "f"((float)bw));
          const int ly = (int)(((float)local + 0.5f) * rbw);
          const int lx = local - ly * bw;
          const int pxl = (int)(b & 0xffu) + lx, pyl = (int)((b >> 8) & 0xffu) + ly;
          const Rec R{sg, j};
          const double x0 = R.at(kFXs), x1 = R.at(kFXs + 1), x2 = R.at(kFXs + 2);
          const double y0 = R.at(kFYs), y1 = R.at(kFYs + 1), y2 = R.at(kFYs + 2);
          const uint32_t fl = sflags[j];
          const double px = (double)(tx0 + pxl) + 0.5, py = (double)(ty0 + pyl) + 0.5;
          // rasterizer.py:161-162, dX / dY exactly as expand_derived forms them
          const double e0 = __dsub_rn(__dmul_rn(__dsub_rn(x2, x1), __dsub_rn(py, y1)),
                                      __dmul_rn(__dsub_rn(y2, y1), __dsub_rn(px, x1)));
          const double e1 = __dsub_rn(__dmul_rn(__dsub_rn(x0, x2), __dsub_rn(py, y2)),
                                      __dmul_rn(__dsub_rn(y0, y2), __dsub_rn(px, x2)));
          const double e2 = __dsub_rn(__dmul_rn(__dsub_rn(x1, x0), __dsub_rn(py, y0)),
                                      __dmul_rn(__dsub_rn(y1, y0), __dsub_rn(px, x0)));
          if ((e0 > 0.0 || (e0 == 0.0 && (fl & 1u))) && (e1 > 0.0 || (e1 == 0.0 && (fl & 2u))) &&
              (e2 > 0.0 || (e2 == 0.0 && (fl & 4u)))) {
            const int pix = pyl * kTW + pxl;
            const uint32_t idx = atomicAdd(pcnt + pix, 1u);
#if TFB_KEEP_PE
            if (idx < (uint32_t)kPC) pc[idx][pix] = (uint8_t)j;
            if (idx == 0u) {  // used only when this is the pixel's sole candidate
              pe[0][pix] = e0;
              pe[1][pix] = e1;
              pe[2][pix] = e2;
            }
#else
            // the first covering pair also records whether, should it stay the pixel's
            // only one, it wins without divisions (bit 7; record slots are < 128)
            uint32_t v = (uint32_t)j;
            if (idx == 0u && TFB_FIRST_FAST && !o.depth) {
              const double e[3] = {e0, e1, e2};
              if (first_fast(e, sg[kSThr * FS + j])) v |= 0x80u;
            }
            if (idx < (uint32_t)kPC) pc[idx][pix] = (uint8_t)v;
#endif
          }
        }
      }
    }
  }
  __syncthreads();

  // one thread per pixel (NT < kTP: kTP / NT pixels per thread): fold its covering
  // records in ascending key order
  auto fold_pixel = [&](const int pt) {
#define PCJ(i) ((int)(pc[(i)][pt] & 0x7f))
    const int pxl = pt & (kTW - 1), pyl = pt / kTW;
    const int px_i = tx0 + pxl, py_i = ty0 + pyl;
    if (px_i >= W || py_i >= H) return;
    const double px = (double)px_i + 0.5, py = (double)py_i + 0.5;
    const uint32_t cnt = pcnt[pt];
    RSTAT(16 + min(cnt, 15u));
    Fold fd;
    fd.init();
    if (cnt == 1u) {
#if TFB_KEEP_PE
      const int j = pc[0][pt];
      const double e[3] = {pe[0][pt], pe[1][pt], pe[2][pt]};
      const bool fast = TFB_FIRST_FAST && !o.depth && first_fast(e, sg[kSThr * FS + j]);
#else
      const int j = pc[0][pt] & 0x7f;
      const bool fast = (pc[0][pt] & 0x80) != 0;
      double e[3];
      if (!fast) edges_at(Rec{sg, j}, sflags[j], px, py, e);  // the pair phase's values, bit for bit
#endif
      if (o.depth) {
        fd.step_e(Rec{sg, j}, e, j);
      } else if (fast) {
        // One texel per triangle (steps = 1) and no float planes: the sole covering
        // record wins, and u in [0, 1], v in [0, u] give i = min(int(u), 0) = 0,
        // j = min(int(v), 0) = 0 (rasterizer.py:196-198), so the texel is 0 whatever
        // the barycentrics are.  They are finite for a winner: w_k >= 0 with
        // 0 < wsum < inf, and the b rows sum to about wsum / wsum, so b.sum() > 0.
        emit_pixel(sc, o, f, (int64_t)f * W * H + (int64_t)(py_i * W + px_i), (int32_t)(skey[j] >> 1), 0, soff[j]);
        return;
      } else {
        fd.first_e(Rec{sg, j}, e, j);
      }
    } else if (cnt == 2u) {  // both slots known: fold in ascending key order
      int j0 = PCJ(0), j1 = PCJ(1);
      if (skey[j1] < skey[j0]) {
        const int tmp = j0;
        j0 = j1;
        j1 = tmp;
      }
      fd.step(Rec{sg, j0}, sflags[j0], px, py, j0);
      fd.step(Rec{sg, j1}, sflags[j1], px, py, j1);
    } else if (cnt > 2u && cnt <= 4u) {  // 3 or 4 slots known: sort by key (a 4-input network) and fold
      int j0 = PCJ(0), j1 = PCJ(1), j2 = PCJ(2), j3 = cnt > 3u ? PCJ(3) : 0;
      uint32_t k0 = skey[j0], k1 = skey[j1], k2 = skey[j2], k3 = cnt > 3u ? skey[j3] : 0xffffffffu;
      auto cx = [](uint32_t &ka, int &ja, uint32_t &kb, int &jb) {
        if (kb < ka) {
          const uint32_t tk = ka;
          ka = kb;
          kb = tk;
          const int tj = ja;
          ja = jb;
          jb = tj;
        }
      };
      cx(k0, j0, k1, j1);
      cx(k2, j2, k3, j3);
      cx(k0, j0, k2, j2);
      cx(k1, j1, k3, j3);
      cx(k1, j1, k2, j2);
      fd.step(Rec{sg, j0}, sflags[j0], px, py, j0);
      fd.step(Rec{sg, j1}, sflags[j1], px, py, j1);
      fd.step(Rec{sg, j2}, sflags[j2], px, py, j2);
      if (cnt > 3u) fd.step(Rec{sg, j3}, sflags[j3], px, py, j3);
    } else if (cnt > 4u && cnt <= (uint32_t)kPC) {  // 5..8 slots known: ascending selection among them
      int64_t last = -1;
      for (uint32_t k = 0; k < cnt; ++k) {
        uint32_t bk = 0xffffffffu;
        int bj = 0;
        for (uint32_t i = 0; i < cnt; ++i) {
          const int ji = PCJ(i);
          const uint32_t ki = skey[ji];
          if ((int64_t)ki > last && ki < bk) {
            bk = ki;
            bj = ji;
          }
        }
        fd.step(Rec{sg, bj}, sflags[bj], px, py, bj);
        last = bk;
      }
    } else if (cnt > (uint32_t)kPC) {  // deeper stacks: repeated smallest-key selection over the tile's records
      int64_t last = -1;  // key of the last folded record
      for (uint32_t k = 0; k < cnt; ++k) {
        unsigned long long best = ~0ull;
        for (uint32_t i = 0; i < n; ++i) {
          const uint32_t key = skey[i];
          if ((int64_t)key <= last) continue;
          const uint32_t bb = sbox[i];
          const int bx = bb & 0xff, by = (bb >> 8) & 0xff;
          if (pxl < bx || pxl >= bx + (int)((bb >> 16) & 0xff) || pyl < by || pyl >= by + (int)(bb >> 24)) continue;
          const unsigned long long cand = ((unsigned long long)key << 32) | i;
          if (cand >= best) continue;
          double e[3];
          if (edges_at(Rec{sg, (int)i}, sflags[i], px, py, e)) best = cand;
        }
        const int j = (int)(best & 0xffffffffu);
        fd.step(Rec{sg, j}, sflags[j], px, py, j);
        last = (int64_t)(best >> 32);
      }
    }
    const uint32_t flags = fd.win >= 0 ? sflags[fd.win] : 0u;
    const int32_t t = fd.win >= 0 ? (int32_t)(skey[fd.win] >> 1) : -1;
    const int64_t off = fd.win >= 0 ? soff[fd.win] : 0;
    write_pixel(sc, cam, o, f, W, H, px_i, py_i, fd, flags, t, off);
#undef PCJ
  };
  if constexpr (NT == kTP) {
    fold_pixel(tid);
  } else {
#pragma unroll 1
    for (int pt = tid; pt < kTP; pt += NT) fold_pixel(pt);
  }
}

// CTAs per SM the register budget must allow for a tile kernel of NT threads
template <int NT>
constexpr int raster_minb() {
  return NT >= kTP ? TFB_RASTER_MINB : (NT >= 64 ? TFB_RASTER_MINB1 : TFB_RASTER_MINB32);
}

// One CTA of NT threads per tile.  With NT < kTP (the default 64 for 16 x 8 tiles) a
// tile's staging (one record per thread) holds NT records and its shared memory is about
// half the kTP-record layout, so twice the tiles are in flight per SM with the same warp
// count: the latency chain of a tile (bin entry -> records -> staging barrier) is hidden by
// more independent tiles.  Tiles with NT < n <= kTP records go to the tier kernels below,
// larger or overflowed ones to k_raster_big.
template <int NT>
__global__ void __launch_bounds__(NT, raster_minb<NT>()) k_raster(tfb_scene sc, const double *__restrict__ cams, int W,
                                                                  int H, int TX, int ntiles, Work w, Outs o) {
  extern __shared__ __align__(16) unsigned char raster_smem[];
  raster_tile<NT>(sc, cams, W, H, TX, ntiles, w, o, blockIdx.z, blockIdx.x, blockIdx.y, raster_smem);
}

// The wider tiers: the tiles a narrower k_raster passed on (n <= 64 records for NT = 64,
// n <= kTP for NT = kTP), NT threads each, a persistent grid walking the tier's list.
template <int NT>
__global__ void __launch_bounds__(NT, raster_minb<NT>()) k_raster_tier(tfb_scene sc, const double *__restrict__ cams,
                                                                       int W, int H, int TX, int ntiles, Work w,
                                                                       Outs o) {
  extern __shared__ __align__(16) unsigned char raster_smem[];
  constexpr int tier = NT >= kTP ? 1 : 0;
  const uint32_t cnt = w.tcnt[tier];
  const uint32_t *list = w.tl + tier * w.tlcap;
  for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    __syncthreads();  // the previous tile's fold is done with the shared memory
    const uint32_t code = list[i];
    const int f = (int)(code / (uint32_t)ntiles), tile = (int)(code % (uint32_t)ntiles);
    raster_tile<NT>(sc, cams, W, H, TX, ntiles, w, o, f, tile % TX, tile / TX, raster_smem);
  }
}

// Tiles with more than kTP records, or whose bin overflowed (then every
// allocated record slot of the frame is scanned; unused slots carry an empty
// bbox).  Records stream through shared memory in chunks in arbitrary order;
// each pixel keeps the kCand smallest covering keys above `lo`, folds them in
// ascending order and repeats with `lo` past the last folded key until no
// covering record is left — the same sequential fold.
__global__ void __launch_bounds__(kTP) k_raster_big(tfb_scene sc, const double *__restrict__ cams, int W,
                                                            int H, int TX, int ntiles, Work w, Outs o) {
  __shared__ RecGeom sgeom[kTP];
  __shared__ RecMeta smeta[kTP];
  __shared__ uint32_t skey[kTP];
  __shared__ uint32_t sidx[kTP];
  __shared__ Cam cam;
  const uint32_t nbig = w.fcnt[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
    const uint32_t code = w.big[bi];
    const int f = (int)(code / ntiles), tile = (int)(code % ntiles);
    const int tx = tile % TX, ty = tile / TX;
    const int wx0 = tx * kTW + (warp % (kTW / 8)) * 8, wy0 = ty * kTH + (warp / (kTW / 8)) * 4;
    const int px_i = wx0 + (lane & 7), py_i = wy0 + (lane >> 3);
    const bool in_img = px_i < W && py_i < H;
    const double px = (double)px_i + 0.5, py = (double)py_i + 0.5;
    __syncthreads();
    load_cam(cam, cams, f);
    const uint32_t tcount = w.tile_count[(int64_t)f * ntiles + tile];
    const bool ovf = tcount > (uint64_t)w.bincap;
    const uint32_t *list = w.list + ((int64_t)f * ntiles + tile) * w.bincap;
    // overflow: every written record slot, [0, nA) and [2(m - nB), 2m)
    const uint32_t na = w.fcnt[4 * f + 2], nb2 = 2u * w.fcnt[4 * f + 3];
    const uint32_t nsrc = ovf ? na + nb2 : tcount;
    const uint32_t clip0 = (uint32_t)(w.rs - nb2);
    const RecStore *recs = w.rec + (int64_t)f * w.rs;

    Fold fd;
    fd.init();
    uint32_t lo = 0;     // next key to consider
    bool need = in_img;  // this pixel still has unfolded candidates
    for (;;) {
      unsigned long long ck[kCand];  // (key << 32) | record index, ascending
#pragma unroll
      for (int i = 0; i < kCand; ++i) ck[i] = ~0ull;
      uint32_t ncand = 0;
      for (uint32_t b0 = 0; b0 < nsrc; b0 += kTP) {
        const uint32_t n = min((uint32_t)kTP, nsrc - b0);
        __syncthreads();
        if (threadIdx.x < n) {
          const uint32_t i = b0 + threadIdx.x;
          const uint32_t r = ovf ? (i < na ? i : clip0 + (i - na)) : list[i];  // holes carry an empty bbox
          sidx[threadIdx.x] = r;
          skey[threadIdx.x] = recs[r].key;
          smeta[threadIdx.x] = recs[r].meta;
          sgeom[threadIdx.x] = expand(recs[r]);
        }
        __syncthreads();
        for (uint32_t j0 = 0; j0 < n; j0 += 32) {
          const uint32_t j = j0 + lane;
          bool rel = false;
          if (j < n) {
            const RecMeta mt = smeta[j];
            rel = mt.x0 <= wx0 + 7 && mt.x1 >= wx0 && mt.y0 <= wy0 + 3 && mt.y1 >= wy0;
          }
          uint32_t m = __ballot_sync(0xffffffffu, rel);
          if (!__any_sync(0xffffffffu, need)) m = 0;
          while (m) {
            const uint32_t jj = j0 + __ffs(m) - 1;
            m &= m - 1;
            const RecMeta mt = smeta[jj];
            if (need && px_i >= mt.x0 && px_i <= mt.x1 && py_i >= mt.y0 && py_i <= mt.y1) {
              const uint32_t key = skey[jj];
              double e[3];
              if (key >= lo && edges_at(AosRec{sgeom + jj}, mt.flags, px, py, e)) {
                ++ncand;
                unsigned long long k = ((unsigned long long)key << 32) | sidx[jj];
#pragma unroll
                for (int i = 0; i < kCand; ++i) {
                  if (k < ck[i]) {
                    const unsigned long long tk = ck[i];
                    ck[i] = k;
                    k = tk;
                  }
                }
              }
            }
          }
        }
      }
      const uint32_t nf = min(ncand, (uint32_t)kCand);
      for (uint32_t i = 0; i < nf; ++i) {
        const uint32_t r = (uint32_t)(ck[i] & 0xffffffffu);
        const RecGeom gk = expand(recs[r]);
        fd.step(AosRec{&gk}, recs[r].meta.flags, px, py, (int32_t)r);
      }
      const bool more = need && ncand > (uint32_t)kCand;
      if (more) lo = (uint32_t)(ck[kCand - 1] >> 32) + 1;
      need = more;
      if (!__syncthreads_or(more)) break;
    }
    if (in_img) {
      const uint32_t flags = fd.win >= 0 ? recs[fd.win].meta.flags : 0u;
      const int32_t t = fd.win >= 0 ? (int32_t)(recs[fd.win].key >> 1) : -1;
      write_pixel(sc, cam, o, f, W, H, px_i, py_i, fd, flags, t, fd.win >= 0 ? recs[fd.win].meta.off : 0);
    }
  }
}

}  // namespace
}  // namespace tfb



using namespace tfb;

extern "C" size_t tfb_raster_workspace_bytes(int64_t num_vertices, int64_t num_triangles, int width, int height,
                                             int max_frames, int64_t pair_capacity) {
  const int TX = (width + kTW - 1) / kTW, TY = (height + kTH - 1) / kTH;
  const int ntiles = TX * TY;
  const int64_t bincap = bin_capacity(pair_capacity, num_triangles, ntiles);
  Work w;
  size_t need = 0;
  carve(nullptr, 0, num_vertices, num_triangles, max_frames, ntiles, bincap, w, &need);
  return need;
}

extern "C" int tfb_rasterize_phases(const tfb_scene *scene, const double *cams, int nframes, int width, int height,
                                    void *workspace, size_t workspace_bytes, int64_t pair_capacity, int32_t *rows_out,
                                    uint32_t *texel_hits, int32_t *tri_out, int32_t *texel_out, double *depth_out,
                                    double *u_out, double *v_out, int phases, void *stream) {
  TFB_REQUIRE(phases >= 1 && phases <= 3, TFB_ERR_VALUE, "tfb_rasterize: phases %d outside 1..3", phases);
  TFB_REQUIRE(scene && cams && rows_out, TFB_ERR_DATA, "tfb_rasterize: null scene, cameras or output");
  TFB_REQUIRE(width > 0 && height > 0 && width < 32768 && height < 32768, TFB_ERR_DATA,
              "tfb_rasterize: image size %dx%d outside 1..32767", width, height);
  TFB_REQUIRE(nframes >= 0, TFB_ERR_DATA, "tfb_rasterize: negative frame count");
  TFB_REQUIRE((tri_out == nullptr) == (texel_out == nullptr), TFB_ERR_VALUE,
              "tfb_rasterize: tri_out and texel_out are given together");
  TFB_REQUIRE((depth_out == nullptr) == (u_out == nullptr) && (u_out == nullptr) == (v_out == nullptr), TFB_ERR_VALUE,
              "tfb_rasterize: depth_out, u_out and v_out are given together");
  TFB_REQUIRE(scene->num_triangles < (1LL << 30), TFB_ERR_CAPACITY,
              "tfb_rasterize: %lld triangles exceed the 2^30 record-key range", (long long)scene->num_triangles);
  TFB_REQUIRE(scene->total_texels < (1LL << 31), TFB_ERR_CAPACITY,
              "tfb_rasterize: %lld texels exceed int32 row ids", (long long)scene->total_texels);
  if (nframes == 0) return TFB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int TX = (width + kTW - 1) / kTW, TY = (height + kTH - 1) / kTH;
  const int ntiles = TX * TY;
  const int64_t m = scene->num_triangles;
  const int64_t bincap = bin_capacity(pair_capacity, m, ntiles);
  Work w;
  size_t need = 0;
  if (!carve(workspace, workspace_bytes, scene->num_vertices, m, nframes, ntiles, bincap, w, &need)) {
    set_error("tfb_rasterize: workspace of %zu bytes is smaller than the %zu required", workspace_bytes, need);
    return TFB_ERR_CAPACITY;
  }
  tfb_scene sc = *scene;
  const bool clustered = sc.num_clusters > 0 && sc.clusters;
  TFB_REQUIRE(!clustered || sc.num_clusters <= w.ncl, TFB_ERR_DATA,
              "tfb_rasterize: %lld clusters for %lld triangles (at most %lld accepted)", (long long)sc.num_clusters,
              (long long)m, (long long)w.ncl);
  if (phases & 1) {  // phase 1: cull, record setup, tile binning (workspace only)
  cudaMemsetAsync(w.fcnt, 0, sizeof(uint32_t) * 4 * (nframes + 1), st);
  cudaMemsetAsync(w.tile_count, 0, sizeof(uint32_t) * ntiles * nframes, st);
  if (m > 0 && clustered) {
    dim3 g0((unsigned)((sc.num_clusters + kThreads - 1) / kThreads), nframes);
    k_ccull<<<g0, kThreads, 0, st>>>(sc, cams, width, height, w);
    // one pass of blocks covers 1/16 of the clusters (a typical view keeps ~1/10);
    // more survivors are strided over
    const int per = TFB_FUSED_SETUP ? kCcsPer : kThreads / kCluster;  // clusters per block
    const int64_t gb = (sc.num_clusters + TFB_CCSETUP_GRID_DIV * per - 1) / (TFB_CCSETUP_GRID_DIV * per);
    dim3 g1((unsigned)(gb < 1 ? 1 : gb), nframes);
    if (TFB_FUSED_SETUP)
      k_ccsetup<<<g1, kCcsPer * kCluster, 0, st>>>(sc, cams, width, height, TX, ntiles, w);
    else
      k_ccands<<<g1, kThreads, 0, st>>>(sc, cams, width, height, w);
  } else if (m > 0) {
    if (sc.num_vertices > 0) {
      dim3 g0((unsigned)((sc.num_vertices + kThreads - 1) / kThreads), nframes);
      k_verts<<<g0, kThreads, 0, st>>>(sc, cams, width, height, w);
    }
    dim3 g1((unsigned)((m + kThreads * kCullPer - 1) / (kThreads * kCullPer)), nframes);
    k_cull<<<g1, kThreads, 0, st>>>(sc, w);
  }
  if (m > 0 && !(clustered && TFB_FUSED_SETUP)) {
    int64_t sb = (m / 3 + kThreads * kSetupPer - 1) / (kThreads * kSetupPer);  // ~1/3 survive a typical cull
    dim3 g2((unsigned)(sb < 1 ? 1 : sb), nframes);
    k_setup<<<g2, kThreads, 0, st>>>(sc, cams, width, height, TX, ntiles, w);
  }
  }
  if (!(phases & 2)) return check_launch("tfb_rasterize");
  // phase 2: the tile kernels over the binned records (reads the workspace phase 1 wrote)
  Outs o{rows_out, texel_hits, tri_out, texel_out, depth_out, u_out, v_out};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  {  // per-device one-time setup; entry points stay re-entrant
    static std::mutex mu;
    static bool smem_set[64] = {};
    static int num_sms[64] = {};
    std::lock_guard<std::mutex> guard(mu);
    auto set_smem = [] {
      cudaFuncSetAttribute(k_raster<kRasterNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(TileSmem<kRasterNT>));
      cudaFuncSetAttribute(k_raster_tier<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem<64>));
      cudaFuncSetAttribute(k_raster_tier<kTP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem<kTP>));
    };
    if (dev >= 0 && dev < 64) {
      if (!smem_set[dev]) {
        set_smem();
        cudaDeviceGetAttribute(&num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
        smem_set[dev] = true;
      }
      sms = num_sms[dev];
    } else {
      set_smem();
    }
  }
  k_raster<kRasterNT><<<dim3(TX, TY, nframes), kRasterNT, sizeof(TileSmem<kRasterNT>), st>>>(sc, cams, width, height,
                                                                                            TX, ntiles, w, o);
  if (kRasterNT < 64)
    k_raster_tier<64><<<sms * raster_minb<64>(), 64, sizeof(TileSmem<64>), st>>>(sc, cams, width, height, TX, ntiles,
                                                                                w, o);
  if (kRasterNT < kTP)
    k_raster_tier<kTP><<<sms * raster_minb<kTP>(), kTP, sizeof(TileSmem<kTP>), st>>>(sc, cams, width, height, TX,
                                                                                    ntiles, w, o);
  k_raster_big<<<sms * (256 / kTP), kTP, 0, st>>>(sc, cams, width, height, TX, ntiles, w, o);
  return check_launch("tfb_rasterize");
}

extern "C" int tfb_rasterize(const tfb_scene *scene, const double *cams, int nframes, int width, int height,
                             void *workspace, size_t workspace_bytes, int64_t pair_capacity, int32_t *rows_out,
                             uint32_t *texel_hits, int32_t *tri_out, int32_t *texel_out, double *depth_out,
                             double *u_out, double *v_out, void *stream) {
  return tfb_rasterize_phases(scene, cams, nframes, width, height, workspace, workspace_bytes, pair_capacity,
                              rows_out, texel_hits, tri_out, texel_out, depth_out, u_out, v_out, 3, stream);
}

#ifdef TFB_RASTER_STATS
extern "C" int tfb_debug_raster_stats(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_rstats, sizeof(g_rstats));
  if (reset) {
    static unsigned long long zero[64] = {0};
    cudaMemcpyToSymbol(g_rstats, zero, sizeof(zero));
  }
  return 0;
}
#endif
