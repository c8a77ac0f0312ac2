// Worst-case projected pixel area per triangle over a set of frames
// (geometry.py:312-380, compute_worst_case_areas) — the pre-pass that sizes
// the texel layout (build_texel_layout, geometry.py:257-291).
//
// One thread per (frame, triangle): FMA-ordered camera transform (as in the
// rasterizer), Sutherland–Hodgman clip against z >= NEAR_PLANE in camera
// space (_clip_polygon with dist = z - NEAR_PLANE), projection, the four image
// edge clips in the reference's order and conditions, then the shoelace area
// 0.5*|dot(x, roll(y,-1)) - dot(y, roll(x,-1))|.  NumPy evaluates those
// short dots through OpenBLAS ddot's non-unit-stride path (x is a stride-2
// view of the (n, 2) polygon), reproduced below operation for operation
// (pinned by the cfg1 golden areas).  The maximum over frames is an
// atomicMax on the IEEE bit pattern (non-negative doubles order as u64).
// Compiled with -fmad=false; FMAs appear only where the reference has them.
#include <math.h>

#include "common.cuh"

namespace tfb {
namespace {

constexpr int kMaxPoly = 10;

struct Cam {
  double R[9], T[3], fx, fy, cx, cy;
};

// _clip_polygon(points, dist), geometry.py:312-326, D-dimensional points
template <int D>
__device__ int clip_poly(const double (*pts)[D], const double *dist, int k, double (*out)[D]) {
  int n = 0;
  for (int i = 0; i < k; ++i) {
    const int j = (i + 1) % k;
    const double di = dist[i], dj = dist[j];
    if (di >= 0) {
#pragma unroll
      for (int q = 0; q < D; ++q) out[n][q] = pts[i][q];
      ++n;
    }
    if ((di >= 0) != (dj >= 0)) {
      const double t = __ddiv_rn(di, __dsub_rn(di, dj));
#pragma unroll
      for (int q = 0; q < D; ++q) out[n][q] = __dadd_rn(pts[i][q], __dmul_rn(t, __dsub_rn(pts[j][q], pts[i][q])));
      ++n;
    }
  }
  return n < 3 ? 0 : n;
}

// OpenBLAS ddot on a stride-2 view (poly[:, 0]): blocks of four accumulate
// t1 += fma(a0,b0,a2*b2), t2 += fma(a1,b1,a3*b3), an FMA tail goes into t1,
// and the result is t1 + t2.
__device__ double blas_ddot_strided(const double (*p)[2], int ca, int cb, int n) {
  double t1 = 0.0, t2 = 0.0;
  int i = 0;
  const int n1 = n & ~3;
  for (; i < n1; i += 4) {
    t1 = __dadd_rn(t1, __fma_rn(p[i][ca], p[(i + 1) % n][cb], __dmul_rn(p[i + 2][ca], p[(i + 3) % n][cb])));
    t2 = __dadd_rn(t2, __fma_rn(p[i + 1][ca], p[(i + 2) % n][cb], __dmul_rn(p[i + 3][ca], p[(i + 4) % n][cb])));
  }
  for (; i < n; ++i) t1 = __fma_rn(p[i][ca], p[(i + 1) % n][cb], t1);
  return __dadd_rn(t1, t2);
}

__device__ double shoelace(const double (*p)[2], int n) {
  // 0.5 * abs(dot(x, roll(y,-1)) - dot(y, roll(x,-1))), geometry.py:329-333
  if (n < 3) return 0.0;
  return __dmul_rn(0.5, fabs(__dsub_rn(blas_ddot_strided(p, 0, 1, n), blas_ddot_strided(p, 1, 0, n))));
}

__device__ double projected_area(const Cam &cam, double W, double H, double P[3][3]) {
  // geometry.py:336-357
  double poly[kMaxPoly][3];
  int k = 3;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int q = 0; q < 3; ++q) poly[i][q] = P[i][q];
  const double zmin = fmin(fmin(P[0][2], P[1][2]), P[2][2]);
  if (zmin < kNearPlane) {
    double dist[3], tmp[kMaxPoly][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dist[i] = __dsub_rn(P[i][2], kNearPlane);
    k = clip_poly<3>(poly, dist, 3, tmp);
    if (k < 3) return 0.0;
    for (int i = 0; i < k; ++i)
#pragma unroll
      for (int q = 0; q < 3; ++q) poly[i][q] = tmp[i][q];
  }
  double a[kMaxPoly][2], b[kMaxPoly][2];
  double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
  for (int i = 0; i < k; ++i) {
    a[i][0] = __dadd_rn(__dmul_rn(__ddiv_rn(poly[i][0], poly[i][2]), cam.fx), cam.cx);
    a[i][1] = __dadd_rn(__dmul_rn(__ddiv_rn(poly[i][1], poly[i][2]), cam.fy), cam.cy);
    xmin = fmin(xmin, a[i][0]);
    xmax = fmax(xmax, a[i][0]);
    ymin = fmin(ymin, a[i][1]);
    ymax = fmax(ymax, a[i][1]);
  }
  if (xmax <= 0 || xmin >= W || ymax <= 0 || ymin >= H) return 0.0;
  double dist[kMaxPoly];
  double(*cur)[2] = a;
  double(*nxt)[2] = b;
  int n = k;
  if (xmin < 0) {
    for (int i = 0; i < n; ++i) dist[i] = cur[i][0];
    n = clip_poly<2>(cur, dist, n, nxt);
    double(*t)[2] = cur; cur = nxt; nxt = t;
  }
  if (n >= 3) {
    double mx = -INFINITY;
    for (int i = 0; i < n; ++i) mx = fmax(mx, cur[i][0]);
    if (mx > W) {
      for (int i = 0; i < n; ++i) dist[i] = __dsub_rn(W, cur[i][0]);
      n = clip_poly<2>(cur, dist, n, nxt);
      double(*t)[2] = cur; cur = nxt; nxt = t;
    }
  }
  if (n >= 3) {
    double mn = INFINITY;
    for (int i = 0; i < n; ++i) mn = fmin(mn, cur[i][1]);
    if (mn < 0) {
      for (int i = 0; i < n; ++i) dist[i] = cur[i][1];
      n = clip_poly<2>(cur, dist, n, nxt);
      double(*t)[2] = cur; cur = nxt; nxt = t;
    }
  }
  if (n >= 3) {
    double mx = -INFINITY;
    for (int i = 0; i < n; ++i) mx = fmax(mx, cur[i][1]);
    if (mx > H) {
      for (int i = 0; i < n; ++i) dist[i] = __dsub_rn(H, cur[i][1]);
      n = clip_poly<2>(cur, dist, n, nxt);
      double(*t)[2] = cur; cur = nxt; nxt = t;
    }
  }
  return shoelace(cur, n);
}

__global__ void __launch_bounds__(256) k_areas(tfb_scene sc, const double *__restrict__ cams, const int32_t *wh,
                                               unsigned long long *areas) {
  const int f = blockIdx.y;
  __shared__ Cam cam;
  if (threadIdx.x < 16) reinterpret_cast<double *>(&cam)[threadIdx.x] = cams[(int64_t)f * 16 + threadIdx.x];
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sc.num_triangles) return;
  double P[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int64_t vi = __ldg(sc.triangles + 3 * t + k);
    const double *v = sc.vertices + 3 * vi;
    const double x = __ldg(v), y = __ldg(v + 1), z = __ldg(v + 2);
#pragma unroll
    for (int r = 0; r < 3; ++r)
      P[k][r] = __dadd_rn(__fma_rn(z, cam.R[3 * r + 2], __fma_rn(y, cam.R[3 * r + 1], __dmul_rn(x, cam.R[3 * r]))),
                          cam.T[r]);
  }
  const double zmax = fmax(fmax(P[0][2], P[1][2]), P[2][2]);
  if (!(zmax >= kNearPlane)) return;  // geometry.py:376
  const double a = projected_area(cam, (double)wh[2 * f], (double)wh[2 * f + 1], P);
  if (a > 0.0) atomicMax(areas + t, (unsigned long long)__double_as_longlong(a));
}

}  // namespace
}  // namespace tfb

using namespace tfb;

extern "C" int tfb_worst_case_areas(const tfb_scene *scene, const double *cams, const int32_t *sizes, int nframes,
                                    double *areas_inout, void *stream) {
  TFB_REQUIRE(scene && cams && sizes && areas_inout, TFB_ERR_DATA, "tfb_worst_case_areas: null argument");
  if (nframes <= 0 || scene->num_triangles <= 0) return TFB_OK;
  dim3 grid((unsigned)((scene->num_triangles + 255) / 256), nframes);
  k_areas<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(*scene, cams, sizes,
                                                               reinterpret_cast<unsigned long long *>(areas_inout));
  return check_launch("tfb_worst_case_areas");
}
