// internal.cuh — structs and host-side entry points shared between the translation units.
#pragma once
#include <nvtx3/nvToolsExt.h>

#include "records.cuh"

// Tracing: every ABI entry point opens an NVTX range on the calling host thread
// (header-only NVTX 3: a no-op unless a tool such as nsys / ncu --nvtx is attached).
struct TsNvtxRange {
  explicit TsNvtxRange(const char* name) { nvtxRangePushA(name); }
  ~TsNvtxRange() { nvtxRangePop(); }
  TsNvtxRange(const TsNvtxRange&) = delete;
  TsNvtxRange& operator=(const TsNvtxRange&) = delete;
};
#define TS_NVTX_CAT2(a, b) a##b
#define TS_NVTX_CAT(a, b) TS_NVTX_CAT2(a, b)
#define TS_NVTX(name) TsNvtxRange TS_NVTX_CAT(ts_nvtx_, __LINE__)(name)

namespace ts {

struct SceneOut {
  int32_t* tet_ids;   // [K]
  int32_t* vert_ids;  // [K,4]
  double* proj;       // [K,4,2]
  double* depths;     // [K,4]
  double* f;          // [K,4]
  double* normals;    // [K,3] (nullable)
  double* md;         // [K]
  double* amax;       // [K] (nullable)
  double* bbox;       // [K,4]
  SplatRec* rec;      // [K]
  int2* prect = nullptr;  // [K] (nullable): the record's packed pixel rectangle (rx, ry) alone
  // [kQBitWords] (nullable, the fused view path): bit qhash(q) set for every splat with a
  // non-empty pixel rectangle (q its 32-bit depth key) — k_bin_count leaves out the splats
  // with an empty rectangle whose depth key no such splat shares (records.cuh)
  uint32_t* qbits = nullptr;
  // never-blend certificate on (records.cuh); off only for the diagnostics flag 128 (the
  // reference's work counts in bench.py's roofline)
  bool certify = true;
};

// host copy of the debug flags (ts_debug_set_flags); bit 128: no never-blend certificate
int ts_impl_debug_flags();

struct BinRec {  // 16 B per splat: first tile and tile-rect extent
  int32_t tx0, ty0, nx, ny;
};

struct BinWork {
  BinRec* br;          // [K]
  uint32_t* q;         // [K]
  int32_t* splat_cnt;  // [K]
  int32_t* tile_cnt;   // [T]  (also the scatter cursor)
  int64_t* scratch;    // scan scratch, compact_blocks(max(K,T))
  int64_t* dev_i64;    // [2]
};

// Caller-owned temporaries of the per-view path (the fused workspace passes its own grow-only
// buffers so no view in flight allocates from the shared stream-ordered pool; nullptr
// members are taken from the pool).
struct ViewScratch {
  int32_t* widx = nullptr;   // [M]   window indices
  double* wz = nullptr;      // [M]   window depths
  int32_t* cnt = nullptr;    // [M]   pairs per list position
  int64_t* scan = nullptr;   // [compact_blocks(M)]
  int32_t* torder = nullptr; // [T]   CTA launch order
  float* rows = nullptr;     // [kGr * M] per-(tile, splat) gradient rows
};

// Sync-free per-view path: device-side counts instead of host round trips.  Buffers are
// sized by host capacities; K = the visible splats (written by the scene build), ovf = set
// when the view needs more than the capacities (every later kernel of the view then exits
// and the caller re-runs the view with larger buffers).
struct Dyn {
  const int64_t* K = nullptr;
  const int* ovf = nullptr;
};

// Deterministic gradient output (fixed point, common.cuh fx_add): when given, the backward
// chain and the regularizers add into these int64 buffers instead of the FP32 d_vert / d_color.
struct Fx {
  long long* vert = nullptr;          // [4 N] (d_sdf, d_deform xyz) * 2^36
  long long* color = nullptr;         // [3 * num_tets] d_color * 2^36 (colour variant)
  unsigned long long* bad = nullptr;  // dropped contributions (non-finite or |v| >= 2^26)
};

struct BinsView {
  const int64_t* starts;
  const int64_t* splat_off;
  const int32_t* items;
  const int32_t* pos_of;
  const uint8_t* nonmono;
  int32_t* witems;  // the compositing lists (k_window_counts)
  int32_t* cpos;    // [M] list position of each compositing-list entry
  int32_t* clen;    // [T] compositing-list length per tile
};

}  // namespace ts

int64_t ts_impl_prefilter(const double* sdf, int R, double s, double thr, int32_t* out_active, int64_t* scratch,
                          cudaStream_t st);
int64_t ts_impl_build_scene(const double* sdf, const double* deform, int R, const ts::Camera& cam, double s,
                            const int32_t* active, int64_t n_active, const ts::SceneOut& out, int64_t* scratch,
                            cudaStream_t st);
// fused view path: scene at the active index (culled tets keep their slot, kCulledRect)
void ts_impl_build_scene_inplace(const double* sdf, const double* deform, int R, const ts::Camera& cam, double s,
                                 const int32_t* active, int64_t n_active, const ts::SceneOut& out, int64_t* n_vis,
                                 cudaStream_t st);
void ts_impl_prepare_records(int64_t K, const double* proj, const double* depths, const double* f,
                             const double* normals, const double* md, const double* bbox, int width, int height,
                             ts::SplatRec* rec, cudaStream_t st);
void ts_impl_bin_count(int64_t K, const double* bbox, const double* md, int tiles_x, int tiles_y, double near_,
                       double far_, const ts::BinWork& w, int64_t* starts, int64_t* splat_off, int64_t* M_out,
                       int64_t* maxL_out, cudaStream_t st, const ts::Dyn* dyn = nullptr,
                       const int2* prect = nullptr, const uint32_t* qbits = nullptr);
void ts_impl_bin_sort(int64_t K, int tiles_x, int tiles_y, const double* md, const ts::BinWork& w,
                      const int64_t* starts, const int64_t* splat_off, int64_t maxL, uint64_t* keys,
                      uint64_t* gscratch, int32_t* items, int32_t* pos_of, uint8_t* nonmono, cudaStream_t st,
                      uint32_t* qsorted = nullptr, const ts::Dyn* dyn = nullptr);
void ts_impl_tile_times(unsigned long long* t2, unsigned int* sm, int n);
int64_t ts_impl_forward_prepare(int tiles_x, int tiles_y, const ts::BinsView& b, int64_t M, const double* md,
                                int n_w, double near_, double far_, const ts::SplatRec* rec, int64_t* item_off,
                                cudaStream_t st, const ts::ViewScratch* scr = nullptr, bool q_ready = false,
                                const ts::Dyn* dyn = nullptr, const int64_t* M_dev = nullptr,
                                const int2* prect = nullptr);
void ts_impl_forward(int tiles_x, int tiles_y, const ts::BinsView& b, const ts::SplatRec* rec, const float* colors,
                     const ts::Scene64& S64, int W, int H, double s, double t_stop, const int64_t* item_off,
                     int64_t n_pairs, uint32_t* pair_bits, float4* pair_rec, float* nmap, float* dmap, float* omap,
                     float* cmap, int32_t* n_proc, int32_t* n_blend, cudaStream_t st,
                     const ts::ViewScratch* scr = nullptr, const ts::Dyn* dyn = nullptr);
void ts_impl_backward(int tiles_x, int tiles_y, const ts::BinsView& b, int64_t M, int64_t K,
                      const ts::SplatRec* rec, const float* colors, const double* fsc, const int32_t* vert_ids,
                      const int32_t* tet_ids, const double* deform, int R, const ts::Camera& cam,
                      const int64_t* item_off, const uint32_t* pair_bits, const float4* pair_rec,
                      const float* maps[4], const float* dmaps[4],
                      const int32_t* n_proc, float* d_vert, float* d_color, cudaStream_t st,
                      const ts::ViewScratch* scr = nullptr, float* status = nullptr,
                      const int32_t* tiles = nullptr, int n_tiles = 0, float* rows_out = nullptr,
                      const ts::Dyn* dyn = nullptr, const ts::Fx* fx = nullptr);
void ts_impl_list_flags(int T, const int64_t* starts, const int32_t* items, const double* md, double near_,
                        double far_, uint8_t* flags, cudaStream_t st);
void ts_impl_saved_records(const int32_t* tiles, int n_tiles, int tiles_x, int W, int H, const ts::BinsView& b,
                           const ts::SplatRec* rec, const int64_t* item_off, const uint32_t* pair_bits,
                           const float4* pair_rec, const int32_t* n_proc, const int64_t* rec_off, int64_t* idx,
                           double* alpha, cudaStream_t st);
void ts_impl_eikonal(const double* sdf, const double* deform, int R, const int32_t* tet_set, int64_t n, float scale,
                     float* d_vert, double* loss, cudaStream_t st, const ts::Fx* fx = nullptr);
void ts_impl_normal_consistency(const double* sdf, const double* deform, int R, float scale, float* d_vert,
                                double* loss, cudaStream_t st, void* scratch = nullptr, const ts::Fx* fx = nullptr,
                                int z0 = 0, int z1 = -1);
void ts_impl_fx_to_f32(const long long* fx, int64_t n, float* out, float* status, cudaStream_t st);
int64_t ts_impl_nc_scratch_bytes(int R);
int ts_impl_mt_count(const double* sdf, const double* deform, int R, int64_t* nv, int64_t* nt, cudaStream_t st);
int ts_impl_mt_run(const double* sdf, const double* deform, int R, void** handle, int64_t* nv, int64_t* nt,
                   cudaStream_t st);
int ts_impl_mt_fetch(void* handle, double* verts, int64_t* tris);
void ts_impl_mt_release(void* handle);
int ts_impl_mt(const double* sdf, const double* deform, int R, double* verts, int64_t* tris, int64_t* nt,
               cudaStream_t st);
void ts_impl_hist(unsigned long long out[32], int reset);
void ts_impl_counters(unsigned long long out[8], int reset);
int ts_impl_rasterize_mesh(const double* verts, int64_t V, const int64_t* tris, int64_t F, const ts::Camera& cam,
                           uint8_t* mask, double* depth, double* normal, cudaStream_t st);
void ts_impl_adam(int64_t N, const float* g4, double* sdf, double* deform, double* m_sdf, double* v_sdf,
                  double* m_def, double* v_def, double lr_sdf, double lr_def, double b1, double b2, int64_t t,
                  double eps, double limit, cudaStream_t st, float* status = nullptr);
void ts_impl_debug_flags(int flags);
void ts_impl_phases(unsigned long long out[16], int reset);
