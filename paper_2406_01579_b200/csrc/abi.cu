// abi.cu — extern "C" entry points (include/tetsplat_b200.h): argument checks, error
// reporting, and dispatch to the kernels in scene.cu / bin.cu / composite.cu /
// regularizers.cu / mt.cu.
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/tetsplat_b200.h"
#include "internal.cuh"
#include "scan.cuh"

using namespace ts;

// ---- error plumbing ------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

void ts_set_error_msg(const char* msg) { g_err = msg; }

static int check_cuda(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? TS_ENOMEM : TS_ECUDA;
  }
  return TS_OK;
}

static Camera to_cam(const ts_camera* c) {
  Camera k;
  memcpy(k.R, c->R, sizeof(k.R));
  memcpy(k.t, c->t, sizeof(k.t));
  k.fx = c->fx; k.fy = c->fy; k.cx = c->cx; k.cy = c->cy;
  k.near_ = c->near_; k.far_ = c->far_;
  k.width = c->width; k.height = c->height;
  return k;
}

// Temporaries come from the device's stream-ordered pool.  Keep freed blocks cached across
// stream synchronisations (the default release threshold of 0 returns them to the driver
// at every sync, turning each per-view scratch allocation into fresh page mappings).
static void keep_pool_warm() {
  static thread_local int dev_done = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_done == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // no hidden cross-stream waits: a stream never reuses another stream's freed block by
    // waiting on it (the views in flight run on separate streams)
    int no = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
  dev_done = dev;
}

template <class T>
static T* dalloc(size_t n, cudaStream_t st) {
  keep_pool_warm();
  T* p = nullptr;
  if (n == 0) n = 1;
  if (cudaMallocAsync(&p, n * sizeof(T), st) != cudaSuccess) return nullptr;
  return p;
}

#define ST(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

const char* ts_last_error(void) { return g_err.c_str(); }
int ts_version(void) { return 1; }

int ts_prefilter(const double* sdf, int32_t R, double s, double thr, int32_t* out, int64_t* count, void* stream) {
  TS_NVTX("ts_prefilter");
  if (!sdf || !out || !count || R < 1) return fail(TS_EINVAL, "ts_prefilter: bad arguments");
  cudaStream_t st = ST(stream);
  const int64_t K = 6ll * R * R * R;
  int64_t* scratch = dalloc<int64_t>(compact_blocks(K), st);
  if (!scratch) return fail(TS_ENOMEM, "ts_prefilter: out of device memory");
  *count = ts_impl_prefilter(sdf, R, s, thr, out, scratch, st);
  cudaFreeAsync(scratch, st);
  return check_cuda("ts_prefilter");
}

int ts_build_scene(const double* sdf, const double* deform, int32_t R, const ts_camera* cam, double s,
                   const int32_t* active, int64_t n_active, const ts_scene* out, int64_t* count, void* stream) {
  TS_NVTX("ts_build_scene");
  if (!sdf || !deform || !cam || !out || !count || R < 1 || n_active < 0 || (n_active > 0 && !active))
    return fail(TS_EINVAL, "ts_build_scene: bad arguments");
  cudaStream_t st = ST(stream);
  int64_t* scratch = dalloc<int64_t>(compact_blocks(n_active, 1), st);
  if (!scratch) return fail(TS_ENOMEM, "ts_build_scene: out of device memory");
  SceneOut o{out->tet_ids, out->vert_ids, out->proj, out->depths, out->f, out->normals, out->mean_depth,
             out->alpha_max, out->bbox, reinterpret_cast<SplatRec*>(out->records)};
  *count = ts_impl_build_scene(sdf, deform, R, to_cam(cam), s, active, n_active, o, scratch, st);
  cudaFreeAsync(scratch, st);
  return check_cuda("ts_build_scene");
}

int ts_prepare_records(const ts_scene* sc, int64_t K, int32_t W, int32_t H, void* stream) {
  TS_NVTX("ts_prepare_records");
  if (!sc || K < 0 || W < 1 || H < 1 || W > 32767 || H > 32767) return fail(TS_EINVAL, "ts_prepare_records: bad arguments");
  ts_impl_prepare_records(K, sc->proj, sc->depths, sc->f, sc->normals, sc->mean_depth, sc->bbox, W, H,
                          reinterpret_cast<SplatRec*>(sc->records), ST(stream));
  return check_cuda("ts_prepare_records");
}

static int tiles_of(const ts_camera* cam, int tile, int& tx, int& ty) {
  if (tile != TS_TILE) return fail(TS_EINVAL, "tile_size must be 16 on the B200 rasterizer");
  if (cam->width < 1 || cam->height < 1 || cam->width > 32767 || cam->height > 32767)
    return fail(TS_EINVAL, "image size must be in [1, 32767]");
  tx = (cam->width + TS_TILE - 1) / TS_TILE;
  ty = (cam->height + TS_TILE - 1) / TS_TILE;
  return TS_OK;
}

int ts_bin_count(const double* bbox, const double* md, int64_t K, const ts_camera* cam, int32_t tile,
                 int64_t* starts, int64_t* splat_off, int64_t* M, int64_t* maxL, void* stream) {
  TS_NVTX("ts_bin_count");
  if (!cam || !starts || !splat_off || !M || !maxL || K < 0 || (K > 0 && (!bbox || !md)))
    return fail(TS_EINVAL, "ts_bin_count: bad arguments");
  int tx, ty;
  if (int e = tiles_of(cam, tile, tx, ty)) return e;
  cudaStream_t st = ST(stream);
  const int64_t T = (int64_t)tx * ty;
  BinWork w;
  w.br = reinterpret_cast<BinRec*>(dalloc<int4>(K, st));
  w.q = dalloc<uint32_t>(K, st);
  w.splat_cnt = dalloc<int32_t>(K, st);
  w.tile_cnt = dalloc<int32_t>(T, st);
  w.scratch = dalloc<int64_t>(compact_blocks(K > T ? K : T), st);
  w.dev_i64 = dalloc<int64_t>(2, st);
  if (!w.br || !w.q || !w.splat_cnt || !w.tile_cnt || !w.scratch || !w.dev_i64)
    return fail(TS_ENOMEM, "ts_bin_count: out of device memory");
  ts_impl_bin_count(K, bbox, md, tx, ty, cam->near_, cam->far_, w, starts, splat_off, M, maxL, st);
  cudaFreeAsync(w.br, st); cudaFreeAsync(w.q, st); cudaFreeAsync(w.splat_cnt, st);
  cudaFreeAsync(w.tile_cnt, st); cudaFreeAsync(w.scratch, st); cudaFreeAsync(w.dev_i64, st);
  return check_cuda("ts_bin_count");
}

int ts_bin_sort(const double* bbox, const double* md, int64_t K, const ts_camera* cam, int32_t tile,
                const ts_bins* b, int64_t M, int64_t maxL, void* stream) {
  TS_NVTX("ts_bin_sort");
  if (!cam || !b || K < 0 || M < 0 || (M > 0 && (!b->items || !b->pos_of || !b->starts || !b->splat_off)) || !b->nonmono)
    return fail(TS_EINVAL, "ts_bin_sort: bad arguments");
  int tx, ty;
  if (int e = tiles_of(cam, tile, tx, ty)) return e;
  cudaStream_t st = ST(stream);
  const int64_t T = (int64_t)tx * ty;
  // recompute per-splat rects/keys (cheap) instead of keeping phase-1 scratch alive
  BinWork w;
  w.br = reinterpret_cast<BinRec*>(dalloc<int4>(K, st));
  w.q = dalloc<uint32_t>(K, st);
  w.splat_cnt = dalloc<int32_t>(K, st);
  w.tile_cnt = dalloc<int32_t>(T, st);
  w.scratch = dalloc<int64_t>(compact_blocks(K > T ? K : T), st);
  w.dev_i64 = dalloc<int64_t>(2, st);
  uint64_t* keys = dalloc<uint64_t>(M, st);
  uint64_t* gs = maxL > 16384 ? dalloc<uint64_t>(2 * M, st) : nullptr;
  if (!w.br || !w.q || !w.splat_cnt || !w.tile_cnt || !w.scratch || !w.dev_i64 || !keys || (maxL > 16384 && !gs))
    return fail(TS_ENOMEM, "ts_bin_sort: out of device memory");
  // phase-1 kernel again for br/q (starts/splat_off are inputs here and are not rewritten)
  int64_t M2 = 0, L2 = 0;
  int64_t* st_tmp = dalloc<int64_t>(T + 1, st);
  int64_t* so_tmp = dalloc<int64_t>(K + 1, st);
  ts_impl_bin_count(K, bbox, md, tx, ty, cam->near_, cam->far_, w, st_tmp, so_tmp, &M2, &L2, st);
  cudaFreeAsync(st_tmp, st);
  cudaFreeAsync(so_tmp, st);
  if (M2 != M) return fail(TS_EINVAL, "ts_bin_sort: M does not match the scene (call ts_bin_count first)");
  ts_impl_bin_sort(K, tx, ty, md, w, b->starts, b->splat_off, maxL, keys, gs, b->items, b->pos_of, b->nonmono, st);
  cudaFreeAsync(w.br, st); cudaFreeAsync(w.q, st); cudaFreeAsync(w.splat_cnt, st);
  cudaFreeAsync(w.tile_cnt, st); cudaFreeAsync(w.scratch, st); cudaFreeAsync(w.dev_i64, st);
  cudaFreeAsync(keys, st);
  if (gs) cudaFreeAsync(gs, st);
  return check_cuda("ts_bin_sort");
}

static Scene64 s64_of(const ts_scene* sc) { return Scene64{sc->proj, sc->depths, sc->f, sc->bbox}; }
// the compositing lists the forward writes and the backward / saved records read
static bool lists_ok(const ts_bins* b, int64_t M) { return M <= 0 || (b->witems && b->cpos && b->clen); }
static BinsView bv_of(const ts_bins* b) {
  return BinsView{b->starts, b->splat_off, b->items, b->pos_of, b->nonmono, b->witems, b->cpos, b->clen};
}

int ts_forward_prepare(const ts_scene* sc, int64_t K, const ts_bins* b, int64_t M, const ts_camera* cam, int32_t n_w,
                       int64_t* item_off, int64_t* out_pairs, void* stream) {
  TS_NVTX("ts_forward_prepare");
  if (n_w < 1) return fail(TS_EINVAL, "resorting window must be >= 1");
  if (!sc || !b || !cam || !item_off || !out_pairs || K < 0 || M < 0)
    return fail(TS_EINVAL, "ts_forward_prepare: bad arguments");
  if (!lists_ok(b, M)) return fail(TS_EINVAL, "ts_forward_prepare: compositing lists (witems / cpos / clen) missing");
  int tx, ty;
  if (int e = tiles_of(cam, TS_TILE, tx, ty)) return e;
  keep_pool_warm();
  *out_pairs = ts_impl_forward_prepare(tx, ty, bv_of(b), M, sc->mean_depth, n_w, cam->near_, cam->far_,
                                       reinterpret_cast<const SplatRec*>(sc->records), item_off, ST(stream));
  return check_cuda("ts_forward_prepare");
}

int ts_render_forward(const ts_scene* sc, int64_t K, const float* colors, const ts_bins* b, int64_t M,
                      const ts_camera* cam, double s, double t_stop, const int64_t* item_off, int64_t n_pairs,
                      uint32_t* pair_bits, void* pair_rec, float* nmap, float* dmap, float* omap, float* cmap,
                      int32_t* n_proc, int32_t* n_blend, void* stream) {
  TS_NVTX("ts_render_forward");
  if (!sc || !b || !cam || !nmap || !dmap || !omap || !n_proc || !n_blend || K < 0 || M < 0 || n_pairs < 0 ||
      (M > 0 && (!item_off || !pair_bits || (n_pairs > 0 && !pair_rec))))
    return fail(TS_EINVAL, "ts_render_forward: bad arguments");
  if (!lists_ok(b, M)) return fail(TS_EINVAL, "ts_render_forward: compositing lists (witems / cpos / clen) missing");
  int tx, ty;
  if (int e = tiles_of(cam, TS_TILE, tx, ty)) return e;
  keep_pool_warm();
  ts_impl_forward(tx, ty, bv_of(b), reinterpret_cast<const SplatRec*>(sc->records), colors, s64_of(sc), cam->width,
                  cam->height, s, t_stop, item_off, n_pairs, pair_bits, reinterpret_cast<float4*>(pair_rec),
                  nmap, dmap, omap, cmap, n_proc, n_blend, ST(stream));
  return check_cuda("ts_render_forward");
}

int ts_render_backward(const ts_scene* sc, int64_t K, const float* colors, const ts_bins* b, int64_t M,
                       const ts_camera* cam, const int64_t* item_off, const uint32_t* pair_bits, const void* pair_rec,
                       const float* const maps[4], const float* const dmaps[4], const int32_t* n_proc,
                       const double* deform, int32_t R, float* d_vert, float* d_color, void* stream) {
  TS_NVTX("ts_render_backward");
  if (!sc || !b || !cam || !maps || !dmaps || !n_proc || !deform || !d_vert || R < 1 || K < 0 || M < 0 ||
      (M > 0 && (!item_off || !pair_bits)))
    return fail(TS_EINVAL, "ts_render_backward: bad arguments");
  if (!lists_ok(b, M)) return fail(TS_EINVAL, "ts_render_backward: compositing lists (witems / cpos / clen) missing");
  for (int i = 0; i < 3; ++i)
    if (!maps[i] || !dmaps[i]) return fail(TS_EINVAL, "ts_render_backward: missing map");
  int tx, ty;
  if (int e = tiles_of(cam, TS_TILE, tx, ty)) return e;
  keep_pool_warm();
  const float* m4[4] = {maps[0], maps[1], maps[2], maps[3]};
  const float* d4[4] = {dmaps[0], dmaps[1], dmaps[2], dmaps[3]};
  ts_impl_backward(tx, ty, bv_of(b), M, K, reinterpret_cast<const SplatRec*>(sc->records), colors, sc->f,
                   sc->vert_ids, sc->tet_ids, deform, R, to_cam(cam), item_off, pair_bits,
                   reinterpret_cast<const float4*>(pair_rec), m4, d4, n_proc, d_vert, d_color, ST(stream));
  return check_cuda("ts_render_backward");
}

// deterministic (fixed-point) outputs: d_vert_fx int64[4N + 1] (entry 4N counts dropped
// contributions), d_color_fx int64[3 * num_tets] (nullable)
static Fx fx_of(int32_t R, int64_t* d_vert_fx, int64_t* d_color_fx) {
  const int64_t n = (int64_t)R + 1;
  Fx fx;
  fx.vert = reinterpret_cast<long long*>(d_vert_fx);
  fx.color = reinterpret_cast<long long*>(d_color_fx);
  fx.bad = reinterpret_cast<unsigned long long*>(d_vert_fx + 4 * n * n * n);
  return fx;
}

int ts_render_backward_fx(const ts_scene* sc, int64_t K, const float* colors, const ts_bins* b, int64_t M,
                          const ts_camera* cam, const int64_t* item_off, const uint32_t* pair_bits,
                          const void* pair_rec, const float* const maps[4], const float* const dmaps[4],
                          const int32_t* n_proc, const double* deform, int32_t R, int64_t* d_vert_fx,
                          int64_t* d_color_fx, void* stream) {
  TS_NVTX("ts_render_backward_fx");
  if (!sc || !b || !cam || !maps || !dmaps || !n_proc || !deform || !d_vert_fx || R < 1 || K < 0 || M < 0 ||
      (M > 0 && (!item_off || !pair_bits)))
    return fail(TS_EINVAL, "ts_render_backward_fx: bad arguments");
  if (!lists_ok(b, M)) return fail(TS_EINVAL, "ts_render_backward_fx: compositing lists (witems / cpos / clen) missing");
  for (int i = 0; i < 3; ++i)
    if (!maps[i] || !dmaps[i]) return fail(TS_EINVAL, "ts_render_backward_fx: missing map");
  int tx, ty;
  if (int e = tiles_of(cam, TS_TILE, tx, ty)) return e;
  keep_pool_warm();
  const float* m4[4] = {maps[0], maps[1], maps[2], maps[3]};
  const float* d4[4] = {dmaps[0], dmaps[1], dmaps[2], dmaps[3]};
  const Fx fx = fx_of(R, d_vert_fx, d_color_fx);
  ts_impl_backward(tx, ty, bv_of(b), M, K, reinterpret_cast<const SplatRec*>(sc->records), colors, sc->f,
                   sc->vert_ids, sc->tet_ids, deform, R, to_cam(cam), item_off, pair_bits,
                   reinterpret_cast<const float4*>(pair_rec), m4, d4, n_proc, nullptr, nullptr, ST(stream), nullptr,
                   nullptr, nullptr, 0, nullptr, nullptr, &fx);
  return check_cuda("ts_render_backward_fx");
}

int ts_bins_from_lists(const int64_t* starts, const int32_t* items, int32_t T, const double* md, double near_,
                       double far_, uint8_t* flags, void* stream) {
  if (!starts || !flags || T < 0 || !(far_ > near_) || (T > 0 && (!items || !md)))
    return fail(TS_EINVAL, "ts_bins_from_lists: bad arguments");
  ts_impl_list_flags(T, starts, items, md, near_, far_, flags, ST(stream));
  return check_cuda("ts_bins_from_lists");
}

int ts_saved_records(const ts_scene* sc, const ts_bins* b, const ts_camera* cam, const int64_t* item_off,
                     const uint32_t* pair_bits, const void* pair_rec, const int32_t* n_proc, const int32_t* tiles,
                     int32_t n_tiles, const int64_t* rec_off, int64_t* idx, double* alpha, void* stream) {
  TS_NVTX("ts_saved_records");
  if (!sc || !b || !cam || !n_proc || n_tiles < 0 || (n_tiles > 0 && (!tiles || !rec_off || !item_off ||
                                                                       !pair_bits || !pair_rec)))
    return fail(TS_EINVAL, "ts_saved_records: bad arguments");
  if (!lists_ok(b, n_tiles)) return fail(TS_EINVAL, "ts_saved_records: compositing lists (witems / cpos / clen) missing");
  int tx, ty;
  if (int e = tiles_of(cam, TS_TILE, tx, ty)) return e;
  ts_impl_saved_records(tiles, n_tiles, tx, cam->width, cam->height, bv_of(b),
                        reinterpret_cast<const SplatRec*>(sc->records), item_off, pair_bits,
                        reinterpret_cast<const float4*>(pair_rec), n_proc, rec_off, idx, alpha, ST(stream));
  return check_cuda("ts_saved_records");
}

int ts_backward_tiles(const ts_scene* sc, int64_t K, const float* colors, const ts_bins* b, int64_t M,
                      const ts_camera* cam, const int64_t* item_off, const uint32_t* pair_bits, const void* pair_rec,
                      const float* const maps[4], const float* const dmaps[4], const int32_t* n_proc,
                      const int32_t* tiles, int32_t n_tiles, float* rows, void* stream) {
  TS_NVTX("ts_backward_tiles");
  if (!sc || !b || !cam || !maps || !dmaps || !n_proc || !rows || K < 0 || M < 0 || n_tiles < 0 ||
      (n_tiles > 0 && !tiles) || (M > 0 && (!item_off || !pair_bits)))
    return fail(TS_EINVAL, "ts_backward_tiles: bad arguments");
  if (!lists_ok(b, M)) return fail(TS_EINVAL, "ts_backward_tiles: compositing lists (witems / cpos / clen) missing");
  for (int i = 0; i < 3; ++i)
    if (!maps[i] || !dmaps[i]) return fail(TS_EINVAL, "ts_backward_tiles: missing map");
  int tx, ty;
  if (int e = tiles_of(cam, TS_TILE, tx, ty)) return e;
  keep_pool_warm();
  const float* m4[4] = {maps[0], maps[1], maps[2], maps[3]};
  const float* d4[4] = {dmaps[0], dmaps[1], dmaps[2], dmaps[3]};
  ts_impl_backward(tx, ty, bv_of(b), M, K, reinterpret_cast<const SplatRec*>(sc->records), colors, sc->f,
                   sc->vert_ids, sc->tet_ids, nullptr, 1, to_cam(cam), item_off, pair_bits,
                   reinterpret_cast<const float4*>(pair_rec), m4, d4, n_proc, nullptr, nullptr, ST(stream), nullptr,
                   nullptr, tiles, n_tiles, rows);
  return check_cuda("ts_backward_tiles");
}

int ts_eikonal(const double* sdf, const double* deform, int32_t R, const int32_t* tet_set, int64_t n, double scale,
               float* d_vert, double* loss, void* stream) {
  TS_NVTX("ts_eikonal");
  if (!sdf || !deform || !d_vert || !loss || R < 1 || n < 0 || (n > 0 && !tet_set))
    return fail(TS_EINVAL, "ts_eikonal: bad arguments");
  ts_impl_eikonal(sdf, deform, R, tet_set, n, (float)scale, d_vert, loss, ST(stream));
  return check_cuda("ts_eikonal");
}

int ts_normal_consistency(const double* sdf, const double* deform, int32_t R, double scale, float* d_vert,
                          double* loss, void* stream) {
  TS_NVTX("ts_normal_consistency");
  if (!sdf || !deform || !d_vert || !loss || R < 1) return fail(TS_EINVAL, "ts_normal_consistency: bad arguments");
  keep_pool_warm();
  ts_impl_normal_consistency(sdf, deform, R, (float)scale, d_vert, loss, ST(stream));
  return check_cuda("ts_normal_consistency");
}

int ts_eikonal_fx(const double* sdf, const double* deform, int32_t R, const int32_t* tet_set, int64_t n,
                  double scale, int64_t* d_vert_fx, double* loss, void* stream) {
  TS_NVTX("ts_eikonal_fx");
  if (!sdf || !deform || !d_vert_fx || !loss || R < 1 || n < 0 || (n > 0 && !tet_set))
    return fail(TS_EINVAL, "ts_eikonal_fx: bad arguments");
  const Fx fx = fx_of(R, d_vert_fx, nullptr);
  ts_impl_eikonal(sdf, deform, R, tet_set, n, (float)scale, nullptr, loss, ST(stream), &fx);
  return check_cuda("ts_eikonal_fx");
}

int ts_normal_consistency_fx(const double* sdf, const double* deform, int32_t R, double scale, int64_t* d_vert_fx,
                             double* loss, void* scratch, void* stream) {
  TS_NVTX("ts_normal_consistency_fx");
  if (!sdf || !deform || !d_vert_fx || !loss || R < 1) return fail(TS_EINVAL, "ts_normal_consistency_fx: bad arguments");
  if (!scratch) keep_pool_warm();
  const Fx fx = fx_of(R, d_vert_fx, nullptr);
  ts_impl_normal_consistency(sdf, deform, R, (float)scale, nullptr, loss, ST(stream), scratch, &fx);
  return check_cuda("ts_normal_consistency_fx");
}

int ts_normal_consistency_slab(const double* sdf, const double* deform, int32_t R, double scale, float* d_vert,
                               int64_t* d_vert_fx, double* loss, void* scratch, int32_t z0, int32_t z1,
                               void* stream) {
  TS_NVTX("ts_normal_consistency_slab");
  if (!sdf || !deform || !loss || R < 1 || (!d_vert == !d_vert_fx) || z0 < 0 || z1 < z0 || z1 > R + 1)
    return fail(TS_EINVAL, "ts_normal_consistency_slab: bad arguments");
  if (!scratch) keep_pool_warm();
  const Fx fx = d_vert_fx ? fx_of(R, d_vert_fx, nullptr) : Fx{};
  ts_impl_normal_consistency(sdf, deform, R, (float)scale, d_vert, loss, ST(stream), scratch,
                             d_vert_fx ? &fx : nullptr, z0, z1);
  return check_cuda("ts_normal_consistency_slab");
}

int ts_fx_to_f32(const int64_t* fx, int64_t n, float* out, float* status, void* stream) {
  if (!fx || !out || n < 0) return fail(TS_EINVAL, "ts_fx_to_f32: bad arguments");
  ts_impl_fx_to_f32(reinterpret_cast<const long long*>(fx), n, out, status, ST(stream));
  return check_cuda("ts_fx_to_f32");
}

int ts_adam_step(int32_t R, const float* d_vert, double* sdf, double* deform, double* m_sdf, double* v_sdf,
                 double* m_def, double* v_def, double lr_sdf, double lr_def, double beta1, double beta2, int64_t t,
                 double eps, double deform_limit, float* status, void* stream) {
  TS_NVTX("ts_adam_step");
  if (!d_vert || !sdf || !deform || !m_sdf || !v_sdf || !m_def || !v_def || R < 1 || t < 1)
    return fail(TS_EINVAL, "ts_adam_step: bad arguments");
  const int64_t n = (int64_t)R + 1;
  ts_impl_adam(n * n * n, d_vert, sdf, deform, m_sdf, v_sdf, m_def, v_def, lr_sdf, lr_def, beta1, beta2, t, eps,
               deform_limit, ST(stream), status);
  return check_cuda("ts_adam_step");
}

int64_t ts_normal_consistency_scratch_bytes(int32_t R) { return R < 1 ? 0 : ts_impl_nc_scratch_bytes(R); }

int ts_normal_consistency_ws(const double* sdf, const double* deform, int32_t R, double scale, float* d_vert,
                             double* loss, void* scratch, void* stream) {
  TS_NVTX("ts_normal_consistency_ws");
  if (!sdf || !deform || !d_vert || !loss || !scratch || R < 1)
    return fail(TS_EINVAL, "ts_normal_consistency_ws: bad arguments");
  ts_impl_normal_consistency(sdf, deform, R, (float)scale, d_vert, loss, ST(stream), scratch);
  return check_cuda("ts_normal_consistency_ws");
}

int ts_marching_tets_count(const double* sdf, const double* deform, int32_t R, int64_t* nv, int64_t* nt,
                           void* stream) {
  keep_pool_warm();
  if (!sdf || !deform || !nv || !nt || R < 1) return fail(TS_EINVAL, "ts_marching_tets_count: bad arguments");
  int rc = ts_impl_mt_count(sdf, deform, R, nv, nt, ST(stream));
  if (rc) return fail(rc, "ts_marching_tets_count failed");
  return check_cuda("ts_marching_tets_count");
}

int ts_marching_tets_run(const double* sdf, const double* deform, int32_t R, void** handle, int64_t* nv,
                         int64_t* nt, void* stream) {
  TS_NVTX("ts_marching_tets_run");
  keep_pool_warm();
  if (!sdf || !deform || !handle || !nv || !nt || R < 1) return fail(TS_EINVAL, "ts_marching_tets_run: bad arguments");
  *handle = nullptr;
  int rc = ts_impl_mt_run(sdf, deform, R, handle, nv, nt, ST(stream));
  if (rc) return fail(rc, "ts_marching_tets_run failed");
  return check_cuda("ts_marching_tets_run");
}

int ts_marching_tets_fetch(void* handle, double* vertices, int64_t* triangles) {
  if (!handle) return fail(TS_EINVAL, "ts_marching_tets_fetch: null handle");
  int rc = ts_impl_mt_fetch(handle, vertices, triangles);
  if (rc) return fail(rc, "ts_marching_tets_fetch failed");
  return check_cuda("ts_marching_tets_fetch");
}

int ts_marching_tets_release(void* handle) {
  ts_impl_mt_release(handle);
  return check_cuda("ts_marching_tets_release");
}

int ts_marching_tets(const double* sdf, const double* deform, int32_t R, double* verts, int64_t* tris,
                     int64_t* nt, void* stream) {
  TS_NVTX("ts_marching_tets");
  keep_pool_warm();
  if (!sdf || !deform || !nt || R < 1) return fail(TS_EINVAL, "ts_marching_tets: bad arguments");
  int rc = ts_impl_mt(sdf, deform, R, verts, tris, nt, ST(stream));
  if (rc) return fail(rc, "ts_marching_tets failed");
  return check_cuda("ts_marching_tets");
}

int ts_rasterize_mesh(const double* vertices, int64_t V, const int64_t* triangles, int64_t F, const ts_camera* cam,
                      uint8_t* mask, double* depth, double* normal, void* stream) {
  TS_NVTX("ts_rasterize_mesh");
  if (!cam || !mask || !depth || !normal || V < 0 || F < 0 || (V > 0 && !vertices) || (F > 0 && !triangles))
    return fail(TS_EINVAL, "ts_rasterize_mesh: bad arguments");
  if (cam->width < 1 || cam->height < 1) return fail(TS_EINVAL, "ts_rasterize_mesh: bad image size");
  keep_pool_warm();
  ts_impl_rasterize_mesh(vertices, V, triangles, F, to_cam(cam), mask, depth, normal, ST(stream));
  return check_cuda("ts_rasterize_mesh");
}

int ts_debug_counters(uint64_t* out8, int reset) {
  if (!out8) return fail(TS_EINVAL, "ts_debug_counters: null output");
  unsigned long long c[8];
  ts_impl_counters(c, reset);
  for (int i = 0; i < 8; ++i) out8[i] = c[i];
  return check_cuda("ts_debug_counters");
}

int ts_debug_hist(uint64_t* out32, int reset) {
  if (!out32) return fail(TS_EINVAL, "ts_debug_hist: null output");
  unsigned long long c[32];
  ts_impl_hist(c, reset);
  for (int i = 0; i < 32; ++i) out32[i] = c[i];
  return check_cuda("ts_debug_hist");
}

int ts_debug_tile_times(uint64_t* t2, uint32_t* sm, int n) {
  if (!t2 || !sm || n < 0 || n > 65536) return fail(TS_EINVAL, "ts_debug_tile_times: bad arguments");
  ts_impl_tile_times(reinterpret_cast<unsigned long long*>(t2), sm, n);
  return check_cuda("ts_debug_tile_times");
}

int ts_debug_phases(uint64_t* out16, int reset) {
  if (!out16) return fail(TS_EINVAL, "ts_debug_phases: null output");
  unsigned long long c[16];
  ts_impl_phases(c, reset);
  for (int i = 0; i < 16; ++i) out16[i] = c[i];
  return check_cuda("ts_debug_phases");
}

int ts_debug_set_flags(int flags) {
  ts_impl_debug_flags(flags);
  return check_cuda("ts_debug_set_flags");
}

}  // extern "C"
