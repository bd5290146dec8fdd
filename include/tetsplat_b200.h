/*
 * tetsplat_b200.h — C ABI of the B200-native TeT-Splatting rasterizer (sm_100a).
 *
 * The drop-in boundary for the reference's kernel plugin (tetsplat.kernels.get_backend(),
 * pkg/src/tetsplat/kernels/__init__.py:35-36; the module paper_2406_01579_b200.kernels binds
 * its five functions) and the per-view
 * orchestration around it (splat.py, raster.py, losses.py, grid.py).  Every pointer
 * argument is a DEVICE pointer unless noted; `stream` is a cudaStream_t (NULL = legacy
 * default stream).  All entry points return 0 on success and a negative TS_E* code on
 * failure; ts_last_error() gives the message (thread-local).  The Python shim maps
 * TS_EINVAL to ValueError and the others to RuntimeError, like the reference.
 *
 * Layouts (row major, C contiguous):
 *   sdf f64[N], deform f64[N,3]       N = (R+1)^3, implicit Kuhn grid of resolution R
 *   gradient buffer f32[N,4]          (d_sdf, d_deform_x, d_deform_y, d_deform_z), ACCUMULATED
 *   scene arrays (capacity >= count)  see ts_scene_t
 *   maps f32: normal [H,W,3], depth [H,W], opacity [H,W], color [H,W,3]
 * Functions that must size their caller-allocated outputs return counts through
 * HOST pointers and synchronise `stream` (marked [sync]).
 */
#ifndef TETSPLAT_B200_H
#define TETSPLAT_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_OK 0
#define TS_EINVAL (-1)  /* invalid argument (ValueError in the shim)     */
#define TS_ENOMEM (-2)  /* device allocation failed                        */
#define TS_ECUDA (-3)   /* CUDA launch / runtime error                     */

/* Pinhole camera (camera.py:13-67): p_cam = R p + t, pixel = (fx X/Z + cx, fy Y/Z + cy). */
typedef struct ts_camera {
  double R[9];
  double t[3];
  double fx, fy, cx, cy, near_, far_;
  int32_t width, height;
  int32_t pad[2];
} ts_camera;

/* SplatScene (splat.py:177-200) in device memory.  `records` is the 96-byte FP32
 * compositing record per splat (derived; see ts_prepare_records). */
typedef struct ts_scene {
  int32_t* tet_ids;   /* [K]     */
  int32_t* vert_ids;  /* [K,4]   */
  double* proj;       /* [K,4,2] */
  double* depths;     /* [K,4]   */
  double* f;          /* [K,4]   */
  double* normals;    /* [K,3]   */
  double* mean_depth; /* [K]     */
  double* alpha_max;  /* [K]     */
  double* bbox;       /* [K,4]   */
  void* records;      /* [K] x 96 B */
} ts_scene;

/* TileBins (raster.py:53-71) plus the B200 extras. */
typedef struct ts_bins {
  int64_t* starts;    /* [T+1]  tile ranges (== reference starts)          */
  int64_t* splat_off; /* [K+1]  exclusive scan of per-splat tile counts     */
  int32_t* items;     /* [M]    splat indices, sorted by (tile, q, index)   */
  int32_t* pos_of;    /* [M]    list position of each (splat, tile) pair     */
  uint8_t* nonmono;   /* [T]    1 when mean depth decreases along the list   */
  int32_t* witems;    /* [M]    compositing lists: the window order without the */
                      /*        entries whose pixel rectangle misses the tile  */
  int32_t* cpos;      /* [M]    list position of each compositing-list entry   */
  int32_t* clen;      /* [T]    compositing-list length per tile               */
} ts_bins;

const char* ts_last_error(void);
int ts_version(void);

/* K1 prefilter (splat.py:66-69): ids of tets with alpha_max >= threshold, increasing.
 * out_active capacity 6 R^3.  [sync] */
int ts_prefilter(const double* sdf, int32_t resolution, double s, double threshold, int32_t* out_active,
                 int64_t* out_count, void* stream);

/* K2 build_scene (splat.py:203-245) for `active` (n_active ids); outputs capacity
 * n_active; out_count = visible splats.  [sync] */
int ts_build_scene(const double* sdf, const double* deform, int32_t resolution, const ts_camera* cam, double s,
                   const int32_t* active, int64_t n_active, const ts_scene* out, int64_t* out_count, void* stream);

/* Compositing records for a scene given only as FP64 arrays (e.g. uploaded). */
int ts_prepare_records(const ts_scene* scene, int64_t K, int32_t width, int32_t height, void* stream);

/* K3/K5 bin_and_sort phase 1 (raster.py:104-131,138-139): starts[T+1], splat_off[K+1];
 * returns M (pairs) and the longest tile list.  tile_size must be 16.  [sync] */
int ts_bin_count(const double* bbox, const double* mean_depth, int64_t K, const ts_camera* cam, int32_t tile_size,
                 int64_t* starts, int64_t* splat_off, int64_t* out_M, int64_t* out_max_len, void* stream);

/* K4 bin_and_sort phase 2 (raster.py:132-141): items/pos_of/nonmono of `bins`. */
int ts_bin_sort(const double* bbox, const double* mean_depth, int64_t K, const ts_camera* cam, int32_t tile_size,
                const ts_bins* bins, int64_t M, int64_t max_len, void* stream);

/* K6 render_forward, step 1 (raster.py:149-156): applies the N_w resorting window to the
 * lists (bins->witems where nonmono) and numbers the view's (pixel, splat) pairs —
 * item_off[M+1] = exclusive scan over list positions of |pixel rectangle ∩ tile|.
 * out_pairs = item_off[M], the size of the pair records below.  [sync] */
int ts_forward_prepare(const ts_scene* scene, int64_t K, const ts_bins* bins, int64_t M, const ts_camera* cam,
                       int32_t n_w, int64_t* item_off, int64_t* out_pairs, void* stream);

/* Words of the pair blend-bit array for P pair records (one spare word for unaligned ORs). */
#define TS_PAIR_BIT_WORDS(n_pairs) (((n_pairs) + 31) / 32 + 1)

/* K6 render_forward, step 2 (forward_tiles _core.pyx:98-229).  colors f32[K,3] / color_map
 * may be NULL.  Pair records (saved state for the backward; P = n_pairs = out_pairs of
 * ts_forward_prepare): pair_bits u32[TS_PAIR_BIT_WORDS(P)] — bit g set when pair g blends
 * (cleared here first) — and pair_rec f32[P,4] written for blending pairs only:
 * (alpha, 1-alpha (negative: clipped at ALPHA_CLIP), s sigmoid(-s f_prev) with the entry
 * face in its two low mantissa bits, s sigmoid(-s f_next) with the exit face likewise).
 * n_proc[H,W]: list entries consumed per pixel; n_blend[H,W]: blended records per pixel
 * (_core.pyx:227-228). */
int ts_render_forward(const ts_scene* scene, int64_t K, const float* colors, const ts_bins* bins, int64_t M,
                      const ts_camera* cam, double s, double t_stop, const int64_t* item_off, int64_t n_pairs,
                      uint32_t* pair_bits, void* pair_rec, float* normal_map, float* depth_map,
                      float* opacity_map, float* color_map, int32_t* n_proc, int32_t* n_blend, void* stream);

/* K7 render_backward (raster.py:206-306 + backward_tiles _core.pyx:344-471): accumulates
 * dL/d(sdf, deform) into d_vert f32[N,4] and dL/dcolor into d_color f32[6R^3,3] (nullable).
 * maps = forward outputs {normal, depth, opacity, color|NULL}; d_maps likewise. */
int ts_render_backward(const ts_scene* scene, int64_t K, const float* colors, const ts_bins* bins, int64_t M,
                       const ts_camera* cam, const int64_t* item_off, const uint32_t* pair_bits,
                       const void* pair_rec, const float* const maps[4], const float* const d_maps[4],
                       const int32_t* n_proc, const double* deform, int32_t resolution, float* d_vert,
                       float* d_color, void* stream);

/* ---- kernel plugin contract (tetsplat.kernels.get_backend(), kernels/__init__.py:35-36) ----
 * Window flags of caller-given tile lists (forward_tiles receives the lists, _core.pyx:98-107):
 * flags[t] = 0 mean depth non-decreasing, 1 sorted by the 32-bit depth key but not by mean
 * depth, 2 not sorted by depth key (the window is replayed over the whole list).  near < far. */
int ts_bins_from_lists(const int64_t* starts, const int32_t* items, int32_t n_tiles, const double* mean_depth,
                       double near_, double far_, uint8_t* flags, void* stream);

/* SavedState.records (_core.pyx:206-209): for each of n_tiles tiles, per pixel (row major in
 * the 16x16 tile) the blended splat indices idx[] and clipped alphas alpha[] in blend order,
 * written from rec_off[i * 256 + pixel] (exclusive scan of the forward's n_blend in that
 * order).  Inputs are a ts_render_forward's bins / pair records / n_proc. */
int ts_saved_records(const ts_scene* scene, const ts_bins* bins, const ts_camera* cam, const int64_t* item_off,
                     const uint32_t* pair_bits, const void* pair_rec, const int32_t* n_proc, const int32_t* tiles,
                     int32_t n_tiles, const int64_t* rec_off, int64_t* idx, double* alpha, void* stream);

/* backward_tiles (_core.pyx:344-471) for n_tiles tiles of a ts_render_forward: the per-splat
 * gradients are ADDED to rows f32[K, 20] (24 with colours): [0,4) d_f, [4,8) d_depths,
 * [8,12) d_proj x, [12,16) d_proj y (per tet vertex), [16,19) d_normals, 19 d_mean_depth,
 * [20,23) d_colors.  No vertex chain (splat_grads_to_vertices stays with the caller). */
int ts_backward_tiles(const ts_scene* scene, int64_t K, const float* colors, const ts_bins* bins, int64_t M,
                      const ts_camera* cam, const int64_t* item_off, const uint32_t* pair_bits, const void* pair_rec,
                      const float* const maps[4], const float* const d_maps[4], const int32_t* n_proc,
                      const int32_t* tiles, int32_t n_tiles, float* rows, void* stream);

/* Fused per-view pipeline over a persistent, grow-only device workspace (one view in flight
 * per workspace).  ts_view_forward = build_scene + bin_and_sort + window + render_forward;
 * out_counts = {K visible splats, M tile pairs, P pixel pairs, longest tile list} (host).  [sync]
 * ts_view_backward = render_backward of the workspace's last forward, accumulated into d_vert
 * (and d_color when the forward had colors_tet f32[6R^3,3]).  status (nullable, device f32):
 * incremented when a map gradient is non-finite (raster.py:209-211 raises ValueError; here the
 * caller raises at its next sync, and ts_adam_step skips the update). */
typedef struct ts_workspace ts_workspace;
ts_workspace* ts_workspace_create(void);
void ts_workspace_destroy(ts_workspace* ws);
int ts_view_forward(ts_workspace* ws, const double* sdf, const double* deform, int32_t resolution,
                    const ts_camera* cam, double s, const int32_t* active, int64_t n_active, int32_t n_w,
                    double t_stop, const float* colors_tet, float* normal_map, float* depth_map, float* opacity_map,
                    float* color_map, int64_t* out_counts, void* stream);
int ts_view_backward(ts_workspace* ws, const double* deform, const float* const maps[4],
                     const float* const d_maps[4], float* d_vert, float* d_color, float* status, void* stream);
const int32_t* ts_view_n_blend(ts_workspace* ws);

/* Deterministic gradients (the reference's fixed-order chunk merge, raster.py:217-247, makes
 * its gradients bitwise reproducible).  The _fx variants add every contribution as the 64-bit
 * integer round(v * 2^36) with integer atomics, so the sums do not depend on the order in
 * which CTAs, streams or (all-reduced as int64) ranks deliver them: d_vert_fx int64[4N + 1]
 * (the interleaved [N,4] layout of d_vert; entry 4N counts contributions dropped because they
 * were non-finite or |v| >= 2^26), d_color_fx int64[3 * 6R^3] (nullable).  Resolution 2^-36.
 * ts_fx_to_f32 converts n entries to FP32 (out[i] = fx[i] * 2^-36) and, when status is given,
 * adds the dropped count fx[n] to status[1] (ts_adam_step then skips the step). */
int ts_view_backward_fx(ts_workspace* ws, const double* deform, const float* const maps[4],
                        const float* const d_maps[4], int64_t* d_vert_fx, int64_t* d_color_fx, float* status,
                        void* stream);
int ts_render_backward_fx(const ts_scene* scene, int64_t K, const float* colors, const ts_bins* bins, int64_t M,
                          const ts_camera* cam, const int64_t* item_off, const uint32_t* pair_bits,
                          const void* pair_rec, const float* const maps[4], const float* const d_maps[4],
                          const int32_t* n_proc, const double* deform, int32_t resolution, int64_t* d_vert_fx,
                          int64_t* d_color_fx, void* stream);
int ts_eikonal_fx(const double* sdf, const double* deform, int32_t resolution, const int32_t* tet_set, int64_t n,
                  double scale, int64_t* d_vert_fx, double* loss, void* stream);
int ts_normal_consistency_fx(const double* sdf, const double* deform, int32_t resolution, double scale,
                             int64_t* d_vert_fx, double* loss, void* scratch, void* stream);
int ts_fx_to_f32(const int64_t* fx, int64_t n, float* out, float* status, void* stream);

/* Normal consistency of one z-slab of vertices (the per-batch regularizer sharded over ranks,
 * SURVEY 8e): adds the gradient of vertex layers z0 <= z < z1 (ids [z0 (R+1)^2, z1 (R+1)^2)) and
 * the penalty of the edges whose lower vertex lies there, computing each pass over the slab plus
 * the halo layers it reads; slabs covering 0..R+1 sum to ts_normal_consistency's result (each
 * vertex's gradient is formed by exactly one slab).  Exactly one of d_vert (f32 [N,4]) and
 * d_vert_fx (fixed point, see ts_view_backward_fx) is given; scratch as for
 * ts_normal_consistency_ws (nullable: stream-ordered allocation); loss is overwritten. */
int ts_normal_consistency_slab(const double* sdf, const double* deform, int32_t resolution, double scale,
                               float* d_vert, int64_t* d_vert_fx, double* loss, void* scratch, int32_t z0,
                               int32_t z1, void* stream);

/* Sync-free per-view path.  With capacities set (cap_M tile pairs, cap_P pixel pairs, cap_L the
 * longest tile list (0 = unbounded); cap_M or cap_P 0 = off)
 * ts_view_forward makes no host round trip: buffers are sized by the capacities (visible
 * splats <= n_active), counts stay on the device and out_counts returns -1.  A view that needs
 * more raises the workspace's overflow flag, which makes every later kernel of the view (and
 * its ts_view_backward) exit; ts_view_status [sync] returns {overflow, K, M, P, max list} of the
 * last forward so the caller can grow the capacities and re-run it; need_out (device int64[5],
 * nullable) receives the same five values stream-ordered, and ts_view_backward of an
 * overflowed view adds 1 to its status[2] (ts_adam_step then skips).  ts_view_need /
 * ts_view_overflow: the device addresses of those counts (int64[4]) and the flag (int32). */
int ts_workspace_set_caps(ts_workspace* ws, int64_t cap_M, int64_t cap_P, int64_t cap_L, int64_t* need_out);
/* stream-ordered: out5 (device int64[5]) = {K, M, P, max list, overflow} of the last forward,
 * and status[2] (device f32, nullable) += 1 when it overflowed (ts_adam_step then skips). */
int ts_view_collect(ts_workspace* ws, float* status, int64_t* out5, void* stream);
int ts_view_status(ts_workspace* ws, int64_t* out5, void* stream);
const int64_t* ts_view_need(ts_workspace* ws);
const int32_t* ts_view_overflow(ts_workspace* ws);

/* K8 eikonal_loss (losses.py:25-36): loss (device f64[1], overwritten) and
 * scale * gradients accumulated into d_vert. */
int ts_eikonal(const double* sdf, const double* deform, int32_t resolution, const int32_t* tet_set, int64_t n,
               double scale, float* d_vert, double* loss, void* stream);

/* K8 normal_consistency_loss (losses.py:39-52), same conventions. */
int ts_normal_consistency(const double* sdf, const double* deform, int32_t resolution, double scale, float* d_vert,
                          double* loss, void* stream);

/* K9 marching_tetrahedra (grid.py:136-239) in one pass: the welded mesh is built into
 * device buffers owned by *out_handle; *out_num_verts / *out_num_tris are its final sizes.
 * Replaces the reference's grid.marching_tetrahedra (grid.py:136) call.  [sync] */
int ts_marching_tets_run(const double* sdf, const double* deform, int32_t resolution, void** out_handle,
                         int64_t* out_num_verts, int64_t* out_num_tris, void* stream);

/* Copy a ts_marching_tets_run result into caller buffers — host or device memory —
 * vertices f64[V,3] (lexicographic (x, y, z)), triangles i64[F,3] (group order of
 * grid.py:192-214, oriented, degenerates removed).  [sync] */
int ts_marching_tets_fetch(void* handle, double* vertices, int64_t* triangles);

/* Free a ts_marching_tets_run result (after any number of fetches). */
int ts_marching_tets_release(void* handle);

/* K9 counts only: the final vertex / triangle counts (capacities for ts_marching_tets).
 * [sync] */
int ts_marching_tets_count(const double* sdf, const double* deform, int32_t resolution, int64_t* out_num_verts,
                           int64_t* out_num_tris, void* stream);

/* K9 into caller device buffers: vertices f64[V,3] (welded, lexicographic (x, y, z)) and
 * triangles i64[F,3] (group order of grid.py:192-214, oriented, degenerates removed);
 * capacities >= ts_marching_tets_count's.  out_counts[0] = F, out_counts[1] = V (host).
 * [sync] */
int ts_marching_tets(const double* sdf, const double* deform, int32_t resolution, double* vertices,
                     int64_t* triangles, int64_t* out_counts, void* stream);

/* ts_normal_consistency with caller-owned scratch (ts_normal_consistency_scratch_bytes(R)
 * bytes of device memory) instead of stream-ordered allocations — for callers that run it
 * beside other streams every step. */
int64_t ts_normal_consistency_scratch_bytes(int32_t resolution);
int ts_normal_consistency_ws(const double* sdf, const double* deform, int32_t resolution, double scale, float* d_vert,
                             double* loss, void* scratch, void* stream);

/* Z-buffered flat-shaded rasterization of a triangle mesh (mesh.py:98-147), the surface-limit
 * reference: vertices f64[V,3], triangles i64[F,3] -> mask u8[H,W], depth f64[H,W] (camera z of
 * the nearest triangle, 0 where uncovered), normal f64[H,W,3] (its unit world face normal).
 * Ties in depth go to the lowest triangle index, like the reference's ordered loop. */
int ts_rasterize_mesh(const double* vertices, int64_t V, const int64_t* triangles, int64_t F, const ts_camera* cam,
                      uint8_t* mask, double* depth, double* normal, void* stream);

/* Adam step of the fit loop (fit.py:70-90) from the interleaved gradient buffer d_vert f32[N,4]:
 * FP64 moments m_sdf, v_sdf [N] and m_def, v_def [N,3], step t >= 1 (bias corrections
 * 1 - beta^t), deformation clamped to +-deform_limit (field.py:40-42) afterwards.
 * status (nullable, device f32[3+]): the non-finite entries of d_vert are counted into
 * status[1] first; when status[0] (non-finite map gradients, ts_view_backward), status[1] or
 * status[2] (a sync-free view overflowed its capacities, ts_view_collect) is non-zero the
 * parameters and moments are left untouched (fit.py:209-212 checks before opt.step) and the
 * caller raises / re-runs at its next sync. */
int ts_adam_step(int32_t resolution, const float* d_vert, double* sdf, double* deform, double* m_sdf,
                 double* v_sdf, double* m_def, double* v_def, double lr_sdf, double lr_def, double beta1,
                 double beta2, int64_t t, double eps, double deform_limit, float* status, void* stream);

/* Diagnostics (since the last reset): out8[0] = (pixel, splat) pairs re-decided in FP64 at
 * a face edge or a degenerate face, out8[1] = pairs re-decided in FP64 at an alpha
 * threshold, out8[2] = forward pairs evaluated, out8[3] = of [0], pairs of splats with a
 * sign-uncertain face determinant; with debug flag 8: out8[4] / out8[5] = of [1], pairs
 * within the f_prev - f_next error bound / near the tiny-alpha or clip bounds, out8[7] =
 * re-decided pairs whose alpha needed the FP64 softplus chain.  [sync] */
int ts_debug_counters(uint64_t* out8, int reset);
/* Diagnostics (debug flag 64): out32[0..16) = alpha re-decisions by floor(-log2(|f_prev - f_next|
 * / bound)), out32[16..32) = edge re-decisions by floor(-log2(|edge value| / band)) (15 = clamp). */
int ts_debug_hist(uint64_t* out32, int reset);

/* Diagnostics for timing experiments only: bit 0 skips the exact FP64 re-decisions
 * (results then no longer match the reference).  Default 0. */
int ts_debug_set_flags(int flags);

/* Diagnostics: with flag bit 1 set, the forward records per-tile start/end %globaltimer
 * (ns) and SM id of its last launch; copies the first n tiles.  [sync] */
int ts_debug_tile_times(uint64_t* t2, uint32_t* sm, int n);

/* Diagnostics: with flag bit 2 set, thread 0 of every compositing CTA sums clock64 cycles
 * between the CTA barriers per phase: out16[0..3] forward stage / A / A' / B,
 * out16[8..12] backward stage / load / B / C / row write (since the last reset).  [sync] */
int ts_debug_phases(uint64_t* out16, int reset);

#ifdef __cplusplus
}
#endif
#endif /* TETSPLAT_B200_H */
