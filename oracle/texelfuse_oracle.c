/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference label-fusion
 * hot path (texelfuse, /root/reference/pkg/src/texelfuse).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load this library, and only as the checker or the CPU baseline; the product
 * (paper_2111_11103_b200) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against fixtures produced by the reference itself (tests/golden/, generated
 * by tests/golden/make_golden.py which imports /root/reference/pkg/src).
 *
 * Arithmetic is IEEE binary64 with no contraction (built with
 * -ffp-contract=off, no -ffast-math) so that every operation rounds exactly
 * where the reference's NumPy expression rounds.  The single exception is the
 * world->camera transform, which the reference evaluates through OpenBLAS
 * dgemm (geometry.py:161); its FMA order  fma(z,R[r][2], fma(y,R[r][1],
 * x*R[r][0])) + t[r]  was verified bit-exact (SURVEY Appendix A1, and
 * tests/test_oracle_golden.py::test_to_camera_bits).
 *
 * Camera packing (16 doubles): R row-major [0..8], t [9..11], fx, fy, cx, cy.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NEAR_PLANE 1e-4 /* geometry.py:26 */
#define DEPTH_TIE 1e-9  /* rasterizer.py:18 */
#define MUL_CLAMP 1e-7  /* fusion.py:39 */

/* geometry.py:159-161 (BLAS FMA order) */
void tfo_to_camera(const double *verts, int64_t n, const double *cam, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    double x = verts[3 * i], y = verts[3 * i + 1], z = verts[3 * i + 2];
    for (int r = 0; r < 3; ++r)
      out[3 * i + r] = fma(z, cam[3 * r + 2], fma(y, cam[3 * r + 1], x * cam[3 * r])) + cam[9 + r];
  }
}

/* NumPy's clip kernel: MIN(MAX(x, lo), hi) with NaN passing through */
static inline double np_max(double a, double b) { return isnan(a) ? a : (a > b ? a : b); }
static inline double np_min(double a, double b) { return isnan(a) ? a : (a < b ? a : b); }

/* rasterizer.py:85-90 */
static int boundary_accept(double ax, double ay, double bx, double by) {
  double dy = by - ay, dx = bx - ax;
  return dy > 0 || (dy == 0 && dx < 0);
}

typedef struct {
  int W, H;
  double fx, fy, cx, cy;
  double *depth;
  int32_t *tri, *texel;
  double *u, *v;
} frame_bufs;

/* rasterizer.py:135-202 — one (sub)triangle; pts are 3 camera-space points,
 * bary the 3x3 barycentric rows of those points in the original triangle. */
static void fill_triangle(frame_bufs *fb, int32_t t, int s, int origin, const double pts[3][3],
                          const double bary_in[3][3]) {
  const int W = fb->W, H = fb->H;
  double xs0[3], ys0[3], zs0[3];
  for (int k = 0; k < 3; ++k) {
    zs0[k] = pts[k][2];
    xs0[k] = pts[k][0] / zs0[k] * fb->fx + fb->cx; /* :138 */
    ys0[k] = pts[k][1] / zs0[k] * fb->fy + fb->cy; /* :139 */
  }
  double xmin = fmin(fmin(xs0[0], xs0[1]), xs0[2]), xmax = fmax(fmax(xs0[0], xs0[1]), xs0[2]);
  double ymin = fmin(fmin(ys0[0], ys0[1]), ys0[2]), ymax = fmax(fmax(ys0[0], ys0[1]), ys0[2]);
  /* :141-146 (clamp in double, then convert: identical to Python int clamp) */
  double x0d = fmax(ceil(xmin - 0.5), 0.0), x1d = fmin(floor(xmax - 0.5), (double)(W - 1));
  double y0d = fmax(ceil(ymin - 0.5), 0.0), y1d = fmin(floor(ymax - 0.5), (double)(H - 1));
  if (!(x0d <= x1d) || !(y0d <= y1d)) return;
  int x0 = (int)x0d, x1 = (int)x1d, y0 = (int)y0d, y1 = (int)y1d;

  double area2 = (xs0[1] - xs0[0]) * (ys0[2] - ys0[0]) - (ys0[1] - ys0[0]) * (xs0[2] - xs0[0]); /* :148 */
  if (area2 == 0.0 || !isfinite(area2)) return;                                             /* :149 */
  int order[3] = {0, 1, 2};
  if (!(area2 > 0)) { order[1] = 2; order[2] = 1; } /* :151 */
  double xs[3], ys[3], zs[3], bary[3][3];
  for (int k = 0; k < 3; ++k) {
    xs[k] = xs0[order[k]]; ys[k] = ys0[order[k]]; zs[k] = zs0[order[k]];
    for (int q = 0; q < 3; ++q) bary[k][q] = bary_in[order[k]][q];
  }
  area2 = fabs(area2);
  int acc[3];
  double dX[3], dY[3];
  for (int k = 0; k < 3; ++k) {
    int a = (k + 1) % 3, b = (k + 2) % 3;
    dX[k] = xs[b] - xs[a];
    dY[k] = ys[b] - ys[a];
    acc[k] = boundary_accept(xs[a], ys[a], xs[b], ys[b]);
  }
  for (int py_i = y0; py_i <= y1; ++py_i) {
    double py = (double)py_i + 0.5;
    for (int px_i = x0; px_i <= x1; ++px_i) {
      double px = (double)px_i + 0.5;
      double e[3];
      int inside = 1;
      for (int k = 0; k < 3; ++k) {
        int a = (k + 1) % 3;
        e[k] = dX[k] * (py - ys[a]) - dY[k] * (px - xs[a]); /* :161 */
        int on = (e[k] > 0) || (e[k] == 0 && acc[k]);        /* :162 */
        inside &= on;
      }
      if (!inside) continue;
      double z = area2 / (e[0] / zs[0] + e[1] / zs[1] + e[2] / zs[2]); /* :170 */
      int64_t pix = (int64_t)py_i * W + px_i;
      if (!(z > 0 && z < fb->depth[pix] - DEPTH_TIE)) continue; /* :171 */
      /* :177-196 perspective-correct barycentric → (u, v) → texel */
      double w0 = e[0] / zs[0], w1 = e[1] / zs[1], w2 = e[2] / zs[2];
      double wsum = w0 + w1 + w2;
      double b[3];
      for (int k = 0; k < 3; ++k) {
        b[k] = (w0 * bary[0][k] + w1 * bary[1][k] + w2 * bary[2][k]) / wsum;
        if (b[k] < 0.0) b[k] = 0.0; /* np.clip(b, 0, None) */
      }
      double bs = b[0] + b[1] + b[2];
      for (int k = 0; k < 3; ++k) b[k] = b[k] / bs;
      double u = 1.0 - b[origin];
      double v = b[(origin + 2) % 3];
      u = np_min(np_max(u, 0.0), 1.0); /* np.clip → umath.clip semantics */
      v = np_min(np_max(v, 0.0), u);
      int64_t i = (int64_t)((double)s * u);
      if (i > s - 1) i = s - 1;
      int64_t j = (int64_t)((double)s * v);
      if (j > i) j = i;
      fb->depth[pix] = z;
      fb->tri[pix] = t;
      fb->texel[pix] = (int32_t)((i * i + i) / 2 + j);
      if (fb->u) fb->u[pix] = u;
      if (fb->v) fb->v[pix] = v;
    }
  }
}

/* rasterizer.py:62-82 — Sutherland–Hodgman against z >= NEAR_PLANE */
static int clip_near(const double pts[3][3], double out_p[4][3], double out_b[4][3]) {
  int n = 0;
  for (int k = 0; k < 3; ++k) {
    const double *a = pts[k], *b = pts[(k + 1) % 3];
    double ba[3] = {0, 0, 0}, bb[3] = {0, 0, 0};
    ba[k] = 1.0;
    bb[(k + 1) % 3] = 1.0;
    int ina = a[2] >= NEAR_PLANE, inb = b[2] >= NEAR_PLANE;
    if (ina) {
      for (int q = 0; q < 3; ++q) { out_p[n][q] = a[q]; out_b[n][q] = ba[q]; }
      ++n;
    }
    if (ina != inb) {
      double tt = (NEAR_PLANE - a[2]) / (b[2] - a[2]);
      for (int q = 0; q < 3; ++q) {
        out_p[n][q] = a[q] + tt * (b[q] - a[q]);
        out_b[n][q] = ba[q] + tt * (bb[q] - ba[q]);
      }
      ++n;
    }
  }
  return n;
}

/* rasterizer.py:93-132.  depth must be provided (H*W doubles); u/v may be NULL.
 * cam_scratch: n*3 doubles or NULL (then allocated). */
int tfo_rasterize(const double *verts, int64_t nv, const int32_t *tris, int64_t m,
                  const int32_t *steps, const int8_t *origins, const double *cam, int W, int H,
                  int32_t *tri_out, int32_t *texel_out, double *depth_out, double *u_out,
                  double *v_out) {
  frame_bufs fb = {W, H, cam[12], cam[13], cam[14], cam[15], depth_out, tri_out, texel_out, u_out, v_out};
  int64_t npx = (int64_t)W * H;
  for (int64_t p = 0; p < npx; ++p) {
    depth_out[p] = INFINITY;
    tri_out[p] = -1;
    texel_out[p] = 0;
    if (u_out) u_out[p] = 0.0;
    if (v_out) v_out[p] = 0.0;
  }
  double *cp = (double *)malloc(sizeof(double) * 3 * (nv > 0 ? nv : 1));
  if (!cp) return 1;
  tfo_to_camera(verts, nv, cam, cp);
  static const double eye[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int64_t t = 0; t < m; ++t) {
    double pts[3][3];
    for (int k = 0; k < 3; ++k)
      for (int q = 0; q < 3; ++q) pts[k][q] = cp[3 * (int64_t)tris[3 * t + k] + q];
    double zmax = fmax(fmax(pts[0][2], pts[1][2]), pts[2][2]);
    double zmin = fmin(fmin(pts[0][2], pts[1][2]), pts[2][2]);
    if (zmax < NEAR_PLANE) continue; /* :111 */
    int s = steps[t], origin = origins[t];
    if (zmin >= NEAR_PLANE) {
      fill_triangle(&fb, (int32_t)t, s, origin, pts, eye);
    } else {
      double pp[4][3], pb[4][3];
      int n = clip_near(pts, pp, pb);
      if (n < 3) continue;
      for (int k = 1; k < n - 1; ++k) { /* fan (0, k, k+1), :119-122 */
        double sp[3][3], sb[3][3];
        int idx[3] = {0, k, k + 1};
        for (int r = 0; r < 3; ++r)
          for (int q = 0; q < 3; ++q) { sp[r][q] = pp[idx[r]][q]; sb[r][q] = pb[idx[r]][q]; }
        fill_triangle(&fb, (int32_t)t, s, origin, sp, sb);
      }
    }
  }
  free(cp);
  return 0;
}

/* ------------------------------------------------------------------------
 * Fusion (fusion.py:114-222) for the CPU baseline.  Frame-parallel over
 * OpenMP threads with private float64 accumulators summed at the end — the
 * monoid fold the reference documents as safe (fusion.py:15-17).
 * agg: 0 sum, 1 maxsum, 2 mul.  wmode: 0 pixels_iid, 1 images_iid, 2 blend.
 * probs[f] points at an (H, W, c) float32 image.  accum (n_x*c) float64 and
 * counts (n_x) int64 are accumulated into (not zeroed).
 * ---------------------------------------------------------------------- */
int tfo_fuse_frames(const double *verts, int64_t nv, const int32_t *tris, int64_t m,
                    const int32_t *steps, const int8_t *origins, const int64_t *offsets,
                    int64_t n_x, int c, const double *cams, int W, int H, int64_t nframes,
                    const float *const *probs, int agg, int wmode, double alpha, double *accum,
                    int64_t *counts, int nthreads) {
  int64_t npx = (int64_t)W * H;
  int err = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
  nthreads = 1;
#endif
  /* private accumulators of every thread, summed row-block-parallel at the end */
  double **accs = (double **)calloc((size_t)nthreads, sizeof(double *));
  int64_t **cnts = (int64_t **)calloc((size_t)nthreads, sizeof(int64_t *));
  if (!accs || !cnts) { free(accs); free(cnts); return 1; }
#pragma omp parallel num_threads(nthreads)
  {
#ifdef _OPENMP
    int me = omp_get_thread_num(), team = omp_get_num_threads();
#else
    int me = 0, team = 1;
#endif
    /* a team of one folds straight into the caller's arrays (no private copy: large layouts) */
    double *acc = team == 1 ? accum : (double *)calloc((size_t)(n_x * c), sizeof(double));
    int64_t *cnt = team == 1 ? counts : (int64_t *)calloc((size_t)n_x, sizeof(int64_t));
    int32_t *frame_cnt = (int32_t *)calloc((size_t)n_x, sizeof(int32_t));
    int32_t *tri = (int32_t *)malloc(sizeof(int32_t) * npx);
    int32_t *tex = (int32_t *)malloc(sizeof(int32_t) * npx);
    double *dep = (double *)malloc(sizeof(double) * npx);
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * npx);
    double *contrib = (double *)malloc(sizeof(double) * c);
    int ok = acc && cnt && frame_cnt && tri && tex && dep && rows && contrib;
    if (!ok) {
#pragma omp atomic write
      err = 1;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t f = 0; f < nframes; ++f) {
      if (!ok) continue;
      tfo_rasterize(verts, nv, tris, m, steps, origins, cams + 16 * f, W, H, tri, tex, dep, NULL, NULL);
      for (int64_t p = 0; p < npx; ++p) {
        rows[p] = tri[p] >= 0 ? offsets[tri[p]] + tex[p] : -1;
        if (rows[p] >= 0) frame_cnt[rows[p]]++;
      }
      const float *pr = probs[f];
      for (int64_t p = 0; p < npx; ++p) {
        int64_t r = rows[p];
        if (r < 0) continue;
        double w = 1.0;
        if (wmode == 1) w = 1.0 / (double)frame_cnt[r];
        else if (wmode == 2) w = (1.0 - alpha) + alpha * (1.0 / (double)frame_cnt[r]);
        const float *pp = pr + p * c;
        if (agg == 0) {
          for (int k = 0; k < c; ++k) acc[r * c + k] += w * (double)pp[k];
        } else if (agg == 1) {
          float mx = pp[0];
          for (int k = 1; k < c; ++k) mx = pp[k] > mx ? pp[k] : mx;
          for (int k = 0; k < c; ++k) acc[r * c + k] += w * (pp[k] == mx ? (double)pp[k] : 0.0);
        } else {
          for (int k = 0; k < c; ++k) {
            double q = (double)pp[k];
            q = q < MUL_CLAMP ? MUL_CLAMP : (q > 1.0 ? 1.0 : q);
            acc[r * c + k] += w * log(q);
          }
        }
        cnt[r]++;
      }
      for (int64_t p = 0; p < npx; ++p)
        if (rows[p] >= 0) frame_cnt[rows[p]] = 0;
    }
    accs[me] = ok ? acc : NULL;
    cnts[me] = ok ? cnt : NULL;
#pragma omp barrier
    /* thread me sums texel rows [lo, hi) over all private accumulators, in thread order */
    int64_t lo = n_x * me / team, hi = n_x * (me + 1) / team;
    for (int q = 0; q < team && team > 1; ++q) {
      if (!accs[q]) continue;
      const double *aq = accs[q];
      const int64_t *cq = cnts[q];
      for (int64_t i = lo * c; i < hi * c; ++i) accum[i] += aq[i];
      for (int64_t i = lo; i < hi; ++i) counts[i] += cq[i];
    }
#pragma omp barrier
    if (team > 1) { free(acc); free(cnt); }
    free(frame_cnt); free(tri); free(tex); free(dep); free(rows); free(contrib);
  }
  free(accs); free(cnts);
  return err;
}

/* fusion.py:186-222 — finalize + argmax.  rows (n_x*c float32) may be NULL. */
void tfo_finalize(const double *accum, const int64_t *counts, int64_t n_x, int c, int agg,
                  float *rows, uint8_t *unobserved, int32_t *labels) {
#pragma omp parallel
  {
  float *tmp = (float *)malloc(sizeof(float) * c);
#pragma omp for schedule(static)
  for (int64_t i = 0; i < n_x; ++i) {
    const double *a = accum + i * c;
    int unobs;
    if (agg == 2) {
      unobs = counts[i] == 0;
      double mx = a[0];
      for (int k = 1; k < c; ++k) mx = a[k] > mx ? a[k] : mx;
      double s = 0;
      for (int k = 0; k < c; ++k) s += exp(a[k] - mx);
      for (int k = 0; k < c; ++k) tmp[k] = (float)(exp(a[k] - mx) / s);
    } else {
      double norm = 0;
      for (int k = 0; k < c; ++k) norm += a[k];
      unobs = counts[i] == 0 || norm <= 0;
      double safe = norm > 0 ? norm : 1.0;
      for (int k = 0; k < c; ++k) tmp[k] = (float)(a[k] / safe);
    }
    if (unobs)
      for (int k = 0; k < c; ++k) tmp[k] = (float)(1.0 / c);
    int best = 0;
    for (int k = 1; k < c; ++k)
      if (tmp[k] > tmp[best]) best = k;
    if (rows) memcpy(rows + i * c, tmp, sizeof(float) * c);
    if (unobserved) unobserved[i] = (uint8_t)unobs;
    labels[i] = unobs ? -1 : best;
  }
  free(tmp);
  }
}

/* ------------------------------------------------------------------------
 * geometry.py:312-380 — worst-case projected area pre-pass.  The shoelace
 * dots (geometry.py:333) go through OpenBLAS ddot's strided path.
 * ---------------------------------------------------------------------- */
static int clip_poly(const double *pts, const double *dist, int k, int D, double *out) {
  int n = 0;
  for (int i = 0; i < k; ++i) {
    int j = (i + 1) % k;
    double di = dist[i], dj = dist[j];
    if (di >= 0) { for (int q = 0; q < D; ++q) out[n * D + q] = pts[i * D + q]; ++n; }
    if ((di >= 0) != (dj >= 0)) {
      double t = di / (di - dj);
      for (int q = 0; q < D; ++q) out[n * D + q] = pts[i * D + q] + t * (pts[j * D + q] - pts[i * D + q]);
      ++n;
    }
  }
  return n < 3 ? 0 : n;
}

/* OpenBLAS ddot, non-unit-stride path (poly[:, 0] is a stride-2 view): blocks
 * of four as t1 += fma(a0,b0,a2*b2), t2 += fma(a1,b1,a3*b3), then an FMA tail
 * into t1, result t1 + t2 — bit-exact against np.dot in this image. */
static double blas_ddot_strided(const double *a, const double *b, int n) {
  double t1 = 0.0, t2 = 0.0;
  int i = 0, n1 = n & -4;
  for (; i < n1; i += 4) {
    t1 += fma(a[i], b[i], a[i + 2] * b[i + 2]);
    t2 += fma(a[i + 1], b[i + 1], a[i + 3] * b[i + 3]);
  }
  for (; i < n; ++i) t1 = fma(a[i], b[i], t1);
  return t1 + t2;
}

static double projected_area(const double *cam, double W, double H, const double P[3][3]) {
  double poly[30], tmp[30], a[20], b[20], dist[10];
  int k = 3;
  for (int i = 0; i < 3; ++i) for (int q = 0; q < 3; ++q) poly[i * 3 + q] = P[i][q];
  double zmin = fmin(fmin(P[0][2], P[1][2]), P[2][2]);
  if (zmin < NEAR_PLANE) {
    for (int i = 0; i < 3; ++i) dist[i] = P[i][2] - NEAR_PLANE;
    k = clip_poly(poly, dist, 3, 3, tmp);
    if (k < 3) return 0.0;
    memcpy(poly, tmp, sizeof(double) * 3 * k);
  }
  double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
  for (int i = 0; i < k; ++i) {
    a[2 * i] = poly[3 * i] / poly[3 * i + 2] * cam[12] + cam[14];
    a[2 * i + 1] = poly[3 * i + 1] / poly[3 * i + 2] * cam[13] + cam[15];
    xmin = fmin(xmin, a[2 * i]); xmax = fmax(xmax, a[2 * i]);
    ymin = fmin(ymin, a[2 * i + 1]); ymax = fmax(ymax, a[2 * i + 1]);
  }
  if (xmax <= 0 || xmin >= W || ymax <= 0 || ymin >= H) return 0.0;
  double *cur = a, *nxt = b, *sw;
  int n = k;
  if (xmin < 0) {
    for (int i = 0; i < n; ++i) dist[i] = cur[2 * i];
    n = clip_poly(cur, dist, n, 2, nxt); sw = cur; cur = nxt; nxt = sw;
  }
  if (n >= 3) {
    double mx = -INFINITY; for (int i = 0; i < n; ++i) mx = fmax(mx, cur[2 * i]);
    if (mx > W) { for (int i = 0; i < n; ++i) dist[i] = W - cur[2 * i];
      n = clip_poly(cur, dist, n, 2, nxt); sw = cur; cur = nxt; nxt = sw; }
  }
  if (n >= 3) {
    double mn = INFINITY; for (int i = 0; i < n; ++i) mn = fmin(mn, cur[2 * i + 1]);
    if (mn < 0) { for (int i = 0; i < n; ++i) dist[i] = cur[2 * i + 1];
      n = clip_poly(cur, dist, n, 2, nxt); sw = cur; cur = nxt; nxt = sw; }
  }
  if (n >= 3) {
    double mx = -INFINITY; for (int i = 0; i < n; ++i) mx = fmax(mx, cur[2 * i + 1]);
    if (mx > H) { for (int i = 0; i < n; ++i) dist[i] = H - cur[2 * i + 1];
      n = clip_poly(cur, dist, n, 2, nxt); sw = cur; cur = nxt; nxt = sw; }
  }
  if (n < 3) return 0.0;
  double xr[10], yr[10], xs[10], ys[10];
  for (int i = 0; i < n; ++i) {
    int j = (i + 1) % n;
    xs[i] = cur[2 * i]; ys[i] = cur[2 * i + 1];
    xr[i] = cur[2 * j]; yr[i] = cur[2 * j + 1];
  }
  return 0.5 * fabs(blas_ddot_strided(xs, yr, n) - blas_ddot_strided(ys, xr, n));
}

void tfo_worst_case_areas(const double *verts, int64_t nv, const int32_t *tris, int64_t m, const double *cams,
                          const int32_t *sizes, int64_t nframes, double *areas) {
  double *cp = (double *)malloc(sizeof(double) * 3 * (nv > 0 ? nv : 1));
  for (int64_t f = 0; f < nframes; ++f) {
    const double *cam = cams + 16 * f;
    tfo_to_camera(verts, nv, cam, cp);
    for (int64_t t = 0; t < m; ++t) {
      double P[3][3];
      for (int k = 0; k < 3; ++k) for (int q = 0; q < 3; ++q) P[k][q] = cp[3 * (int64_t)tris[3 * t + k] + q];
      double zmax = fmax(fmax(P[0][2], P[1][2]), P[2][2]);
      if (!(zmax >= NEAR_PLANE)) continue;
      double a = projected_area(cam, (double)sizes[2 * f], (double)sizes[2 * f + 1], P);
      if (a > areas[t]) areas[t] = a;
    }
  }
  free(cp);
}
