/*
 * texelfuse_b200 — C ABI of the B200-native label-fusion hot path.
 *
 * Drop-in boundary for the reference package texelfuse
 * (/root/reference/pkg/src/texelfuse).  Each entry point replaces the
 * reference function cited beside it; the Python host layer
 * (paper_2111_11103_b200/) keeps the reference's Python API and binds these
 * symbols with ctypes.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (CUDA global memory, allocated
 *    by the caller; the library never allocates or frees on the hot path).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Every call is stream-ordered and asynchronous; no call synchronizes.
 *  - Return value: TFB_OK or one of the TFB_ERR_* codes; tfb_last_error()
 *    returns the message of the last failing call on the calling thread.
 *    The host layer maps codes onto the reference's exception types
 *    (errors.py:4-17): DATA→DataError, CAPACITY→CapacityError,
 *    STATE/CUDA→RuntimeError, VALUE→ValueError.
 *  - Camera packing, 16 float64 per frame: R (3x3 row-major world→camera,
 *    x right / y down / z forward, geometry.py:110-116), t (3), fx, fy, cx, cy.
 *  - A "row" is the global texel index offsets[t] + texel (fusion.py:167);
 *    per-pixel row images use -1 (rasterizer.NONE) for uncovered pixels.
 */
#ifndef TEXELFUSE_B200_H
#define TEXELFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFB_OK 0
#define TFB_ERR_DATA 1     /* DataError     (shape / id / layout mismatch)   */
#define TFB_ERR_CAPACITY 2 /* CapacityError (workspace or smem budget)       */
#define TFB_ERR_STATE 3    /* RuntimeError  (state guard)                    */
#define TFB_ERR_CUDA 4     /* RuntimeError  (CUDA launch / runtime failure)  */
#define TFB_ERR_VALUE 5    /* ValueError    (bad aggregator / mode / alpha)  */

/* fusion.py:34 AGGREGATORS, fusion.py:35 WEIGHT_MODES */
#define TFB_AGG_SUM 0
#define TFB_AGG_MAXSUM 1
#define TFB_AGG_MUL 2
#define TFB_W_PIXELS_IID 0
#define TFB_W_IMAGES_IID 1
#define TFB_W_BLEND 2
#define TFB_W_EXPLICIT 3 /* caller-provided per-pixel weights (fusion.py:145 `weights`) */

/* accumulator element kinds (tfb_fuse / tfb_finalize `accum_kind`) */
#define TFB_ACCUM_F32 0   /* float32: red.global.add.v4.f32, the throughput mode */
#define TFB_ACCUM_F64 1   /* float64: atomicAdd(double), the reference's precision */
#define TFB_ACCUM_FIXED 2 /* int64 fixed point, value * 2^32: integer atomics are order-free, so
                             reruns are bit-identical (the CLI's deterministic=true, SPEC criterion 9) */

/* Mesh + texel layout resident on the device (geometry.py:31-77, 208-232). */
typedef struct tfb_scene {
  const double *vertices;   /* (num_vertices, 3) float64, world metres     */
  const int32_t *triangles; /* (num_triangles, 3) int32                   */
  const int32_t *steps;     /* (num_triangles,) subdivision steps s_t      */
  const int8_t *origins;    /* (num_triangles,) uv-origin vertex 0..2       */
  const int64_t *offsets;   /* (num_triangles,) first global texel row     */
  int64_t num_vertices;
  int64_t num_triangles;
  int64_t total_texels;
  /* Optional spatial clusters for the rasterizer's cluster cull (NULL / 0 =
   * none: every vertex and triangle is tested every frame).  Every triangle
   * must sit in exactly one slot of one cluster.  Results are identical with
   * or without clusters.  At most 2 * ceil(num_triangles / 64) + 1. */
  const struct tfb_cluster *clusters;
  int64_t num_clusters;
} tfb_scene;

/* One cluster: up to 64 triangles and the (at most 128) distinct vertices
 * they use, plus a world-space box containing those vertices. */
typedef struct tfb_cluster {
  int32_t tri[64][4];  /* {triangle id, v0, v1, v2} (vertex ids); id -1 = empty slot */
  uint32_t local[64];  /* corner k of slot i is verts[(local[i] >> 8k) & 0xff]         */
  int32_t nverts;      /* distinct vertices used (<= 128)                             */
  int32_t pad[3];
  int32_t verts[128];  /* their vertex ids                                            */
  double box[6];       /* min x, y, z, max x, y, z                                    */
} tfb_cluster;

const char *tfb_last_error(void);
int tfb_version(void);

/* Tuning knobs (process-wide).  TFB_OPT_FUSE_CTAS_PER_SM caps the resident
 * tfb_fuse CTAs per SM (0 = as many as fit), leaving room for a rasterizer
 * running concurrently on another stream.  TFB_OPT_FUSE_FAST (default 1)
 * enables the specialised float32 / count-weight / c % 4 == 0 scatter-add
 * kernel; 0 routes every tfb_fuse call through the general kernel. */
#define TFB_OPT_FUSE_CTAS_PER_SM 1
#define TFB_OPT_FUSE_FAST 2
int tfb_set_option(int option, int value);

/* Bytes of scratch tfb_rasterize needs for up to `max_frames` frames of
 * width x height (per frame: 2 x num_triangles 96-byte record slots, cull
 * survivors, per-tile counts and fixed-capacity bins of 16x8 tiles).
 * `pair_capacity` = triangle/tile pairs budgeted per frame, spread evenly
 * over the tiles (0 = default: 4 per triangle, at least 512 per tile).
 * Tiles whose bins overflow stay exact through the slow path. */
size_t tfb_raster_workspace_bytes(int64_t num_vertices, int64_t num_triangles, int width, int height,
                                  int max_frames, int64_t pair_capacity);

/* rasterizer.py:93-202 (rasterize) for `nframes` cameras of one size.
 * Bit-exact with the reference: ascending-triangle sequential depth fold
 * with the 1e-9 tie rule, top-left-style edge ownership, near-plane clip +
 * fan, perspective-correct (u, v) → texel id.
 * Outputs (device, nframes*H*W each): rows_out (required).  Optional (NULL
 * to skip), each group all-or-none: tri_out + texel_out (IdImage.triangle /
 * .texel), depth_out + u_out + v_out (IdImage.depth / .u / .v).  texel_hits (nframes*total_texels u32,
 * zeroed by the caller, may be NULL) receives per-frame per-row pixel counts
 * (the np.unique count of fusion.py:135-136). */
int tfb_rasterize(const tfb_scene *scene, const double *cams, int nframes, int width, int height,
                  void *workspace, size_t workspace_bytes, int64_t pair_capacity, int32_t *rows_out,
                  uint32_t *texel_hits, int32_t *tri_out, int32_t *texel_out, double *depth_out,
                  double *u_out, double *v_out, void *stream);

/* tfb_rasterize in two stream-ordered phases (phases = 1, 2 or 3 = both):
 * 1 = cull, record setup and tile binning into the workspace; 2 = the tile
 * kernels that read it and write the outputs.  Both calls take the same
 * arguments; between them the workspace must not be reused.  Lets a caller
 * run batch k+1's phase 1 on a second stream under batch k's scatter-add. */
int tfb_rasterize_phases(const tfb_scene *scene, const double *cams, int nframes, int width, int height,
                         void *workspace, size_t workspace_bytes, int64_t pair_capacity, int32_t *rows_out,
                         uint32_t *texel_hits, int32_t *tri_out, int32_t *texel_out, double *depth_out,
                         double *u_out, double *v_out, int phases, void *stream);

/* rows = offsets[tri] + texel for host-built IdImages (fusion.py:167);
 * -1 where tri == -1.  Out-of-range ids set *bad_flag (device int) to 1. */
int tfb_rows_from_ids(const int32_t *tri, const int32_t *texel, int64_t npix, const tfb_scene *scene,
                      int32_t *rows_out, int32_t *bad_flag, void *stream);

/* Per-frame per-row pixel counts from row images (fusion.py:135-136). */
int tfb_count_hits(const int32_t *rows, int64_t hw, int nframes, int64_t total_texels, uint32_t *hits,
                   void *stream);

/* Zero the hit counters touched by `rows` (leaves the array all-zero again). */
int tfb_clear_hits(const int32_t *rows, int64_t hw, int nframes, int64_t total_texels, uint32_t *hits,
                   void *stream);

/* compute_pixel_weights (fusion.py:114-142) as an (nframes, H*W) float64 image. */
int tfb_pixel_weights(const int32_t *rows, int64_t hw, int nframes, const uint32_t *hits,
                      int64_t total_texels, int weight_mode, double alpha, double *out, void *stream);

/* accumulate_frame (fusion.py:145-183) for `nframes` frames.
 * probs: HOST array of nframes device pointers, each an (H*W, c) float32
 * image; they travel in the kernel parameters (up to 256 frames per launch,
 * more frames split into several launches), so no pointer table is copied and
 * the call is CUDA-graph capturable.  16-byte-aligned maps with float32
 * accumulators and count-derived weights take the specialised kernel; any
 * class count up to ~880 is accepted.  weight_mode TFB_W_EXPLICIT reads `weights`
 * (nframes*H*W float64), the other modes derive w from `texel_hits`.
 * accum: (total_texels, accum_stride) float32 (accum_kind TFB_ACCUM_F32; stride
 * a multiple of 4), float64 (TFB_ACCUM_F64) or int64 fixed point in units of
 * 2^-32 (TFB_ACCUM_FIXED: each piece of equal-row pixels is summed in float64
 * in a fixed order, rounded once and added with an integer atomic, so the
 * result does not depend on scheduling); log-space for TFB_AGG_MUL.
 * counts: (total_texels,) u32 observation counts.  fallback_out (optional,
 * nframes*H*W int32): the per-pixel network argmax probs.argmax(axis=2)
 * (cli.py:293, bindings/__init__.py:112), fused into the same pass. */
int tfb_fuse(const int32_t *rows, int64_t hw, int nframes, const float *const *probs, int num_classes,
             const uint32_t *texel_hits, const double *weights, int64_t total_texels, int aggregator,
             int weight_mode, double alpha, void *accum, int accum_kind, int64_t accum_stride,
             uint32_t *counts, int32_t *fallback_out, void *stream);

/* tfb_fuse with an item order from tfb_fuse_order (NULL: frame-major, as tfb_fuse).
 * The order is honoured by the float32 fast path when the call is one launch
 * (nframes <= 256) and fallback_out is NULL; otherwise every item is processed in
 * frame-major order.  n_items is a DEVICE pointer (written by tfb_fuse_order). */
int tfb_fuse_ordered(const int32_t *rows, int64_t hw, int nframes, const float *const *probs, int num_classes,
                     const uint32_t *texel_hits, const double *weights, int64_t total_texels, int aggregator,
                     int weight_mode, double alpha, void *accum, int accum_kind, int64_t accum_stride,
                     uint32_t *counts, int32_t *fallback_out, const uint32_t *item_order, const uint32_t *n_items,
                     void *stream);

/* Row-block item order for accumulators larger than L2 (configs[3]: 1.73 GB): the
 * (frame, 32-pixel chunk) items of one tfb_fuse launch (nframes <= 256) sorted by
 * the accumulator row block (row >> shift) of their first covered pixel, by a
 * counting sort; chunks with no covered pixel are left out.  The scatter-add then
 * walks the accumulator block by block, so the rows in flight stay in L2 and each
 * is read and written back about once per batch instead of once per frame
 * (fusion.py:180-181 semantics unchanged: the fold is a sum).
 * order_out: nframes*ceil(hw/32) uint32 (frame << 24 | chunk); n_out: one device
 * uint32 (number of items); workspace: tfb_fuse_order_workspace_bytes(). */
size_t tfb_fuse_order_workspace_bytes(int64_t hw, int nframes, int64_t total_texels, int shift);
int tfb_fuse_order(const int32_t *rows, int64_t hw, int nframes, int64_t total_texels, int shift,
                   void *workspace, size_t workspace_bytes, uint32_t *order_out, uint32_t *n_out, void *stream);

/* Test support: y[i] = the float64 natural log the float64-accumulator scatter-add
 * uses (table-driven, csrc/log_f64.cuh) for device arrays x, y of n doubles. */
int tfb_test_log_f64(const double *x, double *y, int64_t n, void *stream);

/* finalize + texel_argmax (fusion.py:186-222).  rows_out (total_texels*c
 * float32), unobserved_out (u8) and labels_out (int32, UNKNOWN = -1) are each
 * optional. */
int tfb_finalize(const void *accum, int accum_kind, int64_t accum_stride, const uint32_t *counts,
                 int64_t total_texels, int num_classes, int aggregator, float *rows_out,
                 uint8_t *unobserved_out, int32_t *labels_out, void *stream);

/* render_labels (renderback.py:28-56): out = labels[row] or -1, then holes
 * filled from `fallback` (nframes*H*W int32, optional). */
int tfb_render(const int32_t *rows, int64_t hw, int nframes, const int32_t *texel_labels,
               int64_t total_texels, const int32_t *fallback, int32_t *out, void *stream);

/* compute_worst_case_areas (geometry.py:360-380): per-triangle maximum
 * projected pixel area over `nframes` cameras, max-folded into areas_inout
 * (num_triangles float64, caller-initialised, normally zeros).  sizes holds
 * (width, height) int32 per frame. */
int tfb_worst_case_areas(const tfb_scene *scene, const double *cams, const int32_t *sizes, int nframes,
                         double *areas_inout, void *stream);

/* probs.argmax(axis=2) (cli.py:293): first maximum, NaN-first like NumPy. */
int tfb_probs_argmax(const float *probs, int64_t npix, int num_classes, int32_t *out, void *stream);

/* SMPB load validation (formats.py:77-93).  out4: 4 doubles of device memory;
 * on completion out4[0] = minimum over all values (NaN if any value is NaN,
 * like np.min) and out4[1] = max over pixels of |sum_k p - 1| with each
 * pixel's sum in float64 in NumPy's pairwise order (NaN if any sum is NaN). */
int tfb_probs_check(const float *probs, int64_t npix, int num_classes, double *out4, void *stream);

/* pixel_accuracy (renderback.py:152-172) for npix label pixels: reference
 * pixels outside [0, c) or flagged in `ignore` (c bytes, may be NULL) are
 * skipped; predictions outside [0, c) count as unknown.  Accumulates (+=)
 * into confusion (c*c u64, row = reference), unknown (c u64) and
 * valid_count (1 u64); the caller zeroes them. */
int tfb_confusion(const int32_t *pred, const int32_t *ref, int64_t npix, int num_classes, const uint8_t *ignore,
                  unsigned long long *confusion, unsigned long long *unknown, unsigned long long *valid_count,
                  void *stream);

/* export_colored_mesh vote (renderback.py:275-294): per triangle the class
 * with the most texels (first maximum wins), -1 when none of its texels has
 * a label in [0, c). */
int tfb_face_majority(const int32_t *texel_labels, const int32_t *steps, const int64_t *offsets,
                      int64_t num_triangles, int num_classes, int32_t *face_class, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TEXELFUSE_B200_H */
