// workspace.cu — fused per-view pipeline over a persistent device workspace.
//
// ts_view_forward  = build_scene (K2) -> bin_and_sort (K3-K5) -> window + pair numbering ->
//                    render_forward (K6), with every intermediate in a workspace whose
//                    buffers only grow.  The three host syncs that size outputs happen inside
//                    C++ (microseconds), not between Python calls.
// ts_view_backward = render_backward (K7) + vertex chain into the shared gradient buffer,
//                    reading the saved state the last ts_view_forward left in the workspace.
// With capacities set (ts_workspace_set_caps) the forward is SYNC-FREE: buffers are sized by
// the capacities (visible splats <= active tets, tile pairs <= cap_M, pixel pairs <= cap_P),
// every count stays on the device (Dyn), and a view that needs more sets the workspace's
// overflow flag — all its later kernels exit, the caller reads ts_view_status at its next
// sync, grows the capacities and re-runs the view.
// The fine-grained entry points in abi.cu stay for reference-style use (and tests).
#include <cstring>

#include "../../include/tetsplat_b200.h"
#include "internal.cuh"
#include "scan.cuh"

using namespace ts;

namespace {

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t n) {
    const size_t bytes = (n ? n : 1) * sizeof(T);
    if (bytes > cap) {
      if (p) cudaFree(p);
      size_t c = bytes + bytes / 4;  // grow with headroom
      if (cudaMalloc(&p, c) != cudaSuccess) {
        p = nullptr;
        cap = 0;
        return nullptr;
      }
      cap = c;
    }
    return reinterpret_cast<T*>(p);
  }
};

}  // namespace

struct ts_workspace {
  // scene
  Buf tet_ids, vert_ids, proj, depths, f, normals, md, amax, bbox, rec, colors, prect, qbits;
  // bins
  Buf starts, items, nonmono, witems, cpos, clen, br, q, splat_cnt, tile_cnt, scratch, dev_i64, keys, gsort;
  // forward state
  Buf item_off, pair_bits, pair_rec, n_proc, n_blend;
  // per-view temporaries (kept so no view in flight allocates from the shared pool)
  Buf widx, wz, pcnt, pscan, torder, rows;
  // sync-free path: capacities (0 = sizing syncs), device counts {K, M, P, maxL} + overflow flag
  Buf need, ovf;
  int64_t capM = 0, capP = 0, capL = 0;
  int64_t* need_out = nullptr;  // caller's device int64[5] receiving {K, M, P, max list, overflow}
  bool dyn = false;
  // view description of the last forward (capacities on the sync-free path)
  int64_t K = 0, M = 0, P = 0, maxL = 0;
  int64_t Kvis = 0;  // visible splats (reported; the fused scene keeps every active tet's slot)
  int tiles_x = 0, tiles_y = 0, R = 0;
  Camera cam{};
  double s = 0.0;
  bool color = false;
  bool valid = false;
};

void ts_set_error_msg(const char* msg);  // abi.cu (ts_last_error)

static int ws_fail(int code, const char* msg) {
  ts_set_error_msg(msg);
  return code;
}

static Camera cam_of(const ts_camera* c) {
  Camera k;
  memcpy(k.R, c->R, sizeof(k.R));
  memcpy(k.t, c->t, sizeof(k.t));
  k.fx = c->fx; k.fy = c->fy; k.cx = c->cx; k.cy = c->cy;
  k.near_ = c->near_; k.far_ = c->far_;
  k.width = c->width; k.height = c->height;
  return k;
}

namespace ts {
__global__ void k_gather_colors(int64_t K, const int32_t* __restrict__ tet_ids, const float* __restrict__ ctet,
                                float* __restrict__ out, const int64_t* __restrict__ Kdev) {
  if (Kdev) K = min(K, *Kdev);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < 3; ++c) out[k * 3 + c] = ctet[(int64_t)tet_ids[k] * 3 + c];
}

// a count the sync-free path produced on the device: recorded, and the overflow flag raised
// when it exceeds its capacity; the last check also copies {K, M, P, max list, overflow} to
// the caller's slot (ts_workspace_set_caps) when there is one
__global__ void k_caps_check(const int64_t* __restrict__ total, int64_t cap, int* __restrict__ ovf,
                             int64_t* __restrict__ need_slot, const int64_t* __restrict__ extra,
                             int64_t* __restrict__ extra_slot, int64_t extra_cap, const int64_t* __restrict__ need,
                             int64_t* __restrict__ out5) {
  const int64_t v = *total;
  *need_slot = v;
  int o = v > cap;
  if (extra) {
    *extra_slot = *extra;
    o |= *extra > extra_cap;
  }
  if (o) atomicOr(ovf, 1);
  if (out5) {
    for (int i = 0; i < 4; ++i) out5[i] = need[i];
    out5[4] = *ovf;
  }
}
}  // namespace ts

extern "C" {

ts_workspace* ts_workspace_create(void) { return new ts_workspace(); }

int ts_workspace_set_caps(ts_workspace* ws, int64_t cap_M, int64_t cap_P, int64_t cap_L, int64_t* need_out) {
  if (!ws || cap_M < 0 || cap_P < 0 || cap_L < 0) return ws_fail(TS_EINVAL, "ts_workspace_set_caps: bad arguments");
  ws->capM = cap_M;
  ws->capP = cap_P;
  ws->capL = cap_L;
  ws->need_out = need_out;
  return TS_OK;
}

int ts_view_status(ts_workspace* ws, int64_t* out5, void* stream) {
  if (!ws || !out5) return ws_fail(TS_EINVAL, "ts_view_status: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!ws->dyn) {
    out5[0] = 0;
    out5[1] = ws->Kvis;
    out5[2] = ws->M;
    out5[3] = ws->P;
    out5[4] = ws->maxL;
    return TS_OK;
  }
  int h = 0;
  int64_t n[4] = {0, 0, 0, 0};
  cudaMemcpyAsync(&h, ws->ovf.p, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(n, ws->need.p, sizeof(n), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return ws_fail(TS_ECUDA, cudaGetErrorString(cudaGetLastError()));
  out5[0] = h;
  for (int i = 0; i < 4; ++i) out5[1 + i] = n[i];
  return TS_OK;
}

__global__ void k_view_collect(const int64_t* __restrict__ need, const int* __restrict__ ovf, float* status,
                               int64_t* __restrict__ out) {
  const int o = ovf ? *ovf : 0;
  if (o && status) atomicAdd(status + 2, 1.0f);
  for (int i = 0; i < 4; ++i) out[i] = need ? need[i] : 0;
  out[4] = o;
}

int ts_view_collect(ts_workspace* ws, float* status, int64_t* out5, void* stream) {
  TS_NVTX("ts_view_collect");
  if (!ws || !out5) return ws_fail(TS_EINVAL, "ts_view_collect: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (ws->dyn)
    k_view_collect<<<1, 1, 0, st>>>(reinterpret_cast<int64_t*>(ws->need.p), reinterpret_cast<int*>(ws->ovf.p), status,
                                    out5);
  else {
    const int64_t h[5] = {ws->Kvis, ws->M, ws->P, ws->maxL, 0};
    cudaMemcpyAsync(out5, h, sizeof(h), cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);  // h is a stack buffer (sizing path: the host already waited)
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : ws_fail(TS_ECUDA, cudaGetErrorString(e));
}

// device pointers of the last forward's {K, M, P, maxL} (int64) and overflow flag (int32)
const int64_t* ts_view_need(ts_workspace* ws) { return ws ? reinterpret_cast<int64_t*>(ws->need.p) : nullptr; }
const int32_t* ts_view_overflow(ts_workspace* ws) { return ws ? reinterpret_cast<int32_t*>(ws->ovf.p) : nullptr; }

void ts_workspace_destroy(ts_workspace* ws) {
  if (!ws) return;
  Buf* all[] = {&ws->prect, &ws->qbits, &ws->need, &ws->ovf, &ws->tet_ids, &ws->vert_ids, &ws->proj, &ws->depths, &ws->f, &ws->normals, &ws->md, &ws->amax,
                &ws->bbox, &ws->rec, &ws->colors, &ws->starts, &ws->items,
                &ws->nonmono, &ws->witems, &ws->cpos, &ws->clen, &ws->br, &ws->q, &ws->splat_cnt, &ws->tile_cnt, &ws->scratch,
                &ws->dev_i64, &ws->keys, &ws->gsort, &ws->item_off, &ws->pair_bits, &ws->pair_rec,
                &ws->n_proc, &ws->widx, &ws->wz, &ws->pcnt, &ws->pscan, &ws->torder, &ws->rows, &ws->n_blend};
  cudaDeviceSynchronize();
  for (Buf* b : all)
    if (b->p) cudaFree(b->p);
  delete ws;
}

// the sync-free forward (see the file comment)
static int view_forward_dyn(ts_workspace* ws, const double* sdf, const double* deform, int32_t R, const Camera& cam,
                            double s, const int32_t* active, int64_t n_active, int32_t n_w, double t_stop,
                            const float* colors_tet, float* nmap, float* dmap, float* omap, float* cmap,
                            int64_t* out_counts, cudaStream_t st) {
  const int tx = (cam.width + TS_TILE - 1) / TS_TILE, ty = (cam.height + TS_TILE - 1) / TS_TILE;
  const int64_t T = (int64_t)tx * ty, HW = (int64_t)cam.width * cam.height;
  const int64_t cap = n_active > 0 ? n_active : 1, capM = ws->capM, capP = ws->capP;
  int64_t* need = ws->need.get<int64_t>(4);
  int* ovf = ws->ovf.get<int>(1);
  SceneOut so{ws->tet_ids.get<int32_t>(cap), ws->vert_ids.get<int32_t>(cap * 4), nullptr,
              nullptr, ws->f.get<double>(cap * 4), nullptr,
              ws->md.get<double>(cap), nullptr, ws->bbox.get<double>(cap * 4),
              ws->rec.get<SplatRec>(cap), ws->prect.get<int2>(cap)};
  const int64_t nmax = cap > T ? (cap > capM ? cap : capM) : (T > capM ? T : capM);
  int64_t* scratch = ws->scratch.get<int64_t>(compact_blocks(nmax + 1, 1));
  so.qbits = reinterpret_cast<uint32_t*>(ws->qbits.get<unsigned char>(kQBytes));
  if (!need || !ovf || !so.tet_ids || !so.rec || !scratch || !so.qbits)
    return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  cudaMemsetAsync(so.qbits, 0, kQBytesZero, st);                                          // keys, max md
  cudaMemsetAsync(reinterpret_cast<unsigned char*>(so.qbits) + kQBytesZero, 0xff, kQBytes - kQBytesZero, st);  // min md
  cudaMemsetAsync(ovf, 0, sizeof(int), st);
  cudaMemsetAsync(need, 0, 4 * sizeof(int64_t), st);
  Dyn dyn;
  dyn.K = nullptr;  // the scene is indexed by active tet: all cap slots are valid (culled ones skipped)
  dyn.ovf = ovf;
  // need[0] receives the visible count (reported only)
  ts_impl_build_scene_inplace(sdf, deform, R, cam, s, active, n_active, so, need, st);
  // ---- bins (capacity-sized, counts on the device) ----------------------------------------
  BinWork w;
  w.br = reinterpret_cast<BinRec*>(ws->br.get<int4>(cap));
  w.q = ws->q.get<uint32_t>(cap);
  w.splat_cnt = ws->splat_cnt.get<int32_t>(cap);
  w.tile_cnt = ws->tile_cnt.get<int32_t>(T);
  w.scratch = scratch;
  w.dev_i64 = ws->dev_i64.get<int64_t>(2);
  int64_t* starts = ws->starts.get<int64_t>(T + 1);
  uint8_t* nonmono = ws->nonmono.get<uint8_t>(T);
  int32_t* items = ws->items.get<int32_t>(capM);
  int32_t* witems = ws->witems.get<int32_t>(capM);
  int32_t* cpos = ws->cpos.get<int32_t>(capM);
  int32_t* clen = ws->clen.get<int32_t>(T);
  uint64_t* keys = ws->keys.get<uint64_t>(capM);
  uint64_t* gs = ws->capL > 16384 || ws->capL == 0 ? ws->gsort.get<uint64_t>(2 * capM) : keys;  // unused <= 16384
  int32_t* pcnt = ws->pcnt.get<int32_t>(capM);
  int64_t* item_off = ws->item_off.get<int64_t>(capM + 1);
  int32_t* n_proc = ws->n_proc.get<int32_t>(HW);
  int32_t* n_blend = ws->n_blend.get<int32_t>(HW);
  ViewScratch scr;
  scr.widx = ws->widx.get<int32_t>(capM);
  scr.wz = ws->wz.get<double>(capM);
  scr.cnt = pcnt;
  scr.scan = ws->pscan.get<int64_t>(compact_blocks(capM));
  scr.torder = ws->torder.get<int32_t>(T);
  scr.rows = ws->rows.get<float>(24 * cap);
  uint32_t* pbits = ws->pair_bits.get<uint32_t>(TS_PAIR_BIT_WORDS(capP));
  float4* prec = ws->pair_rec.get<float4>(capP);
  if (!w.br || !w.q || !w.splat_cnt || !w.tile_cnt || !w.dev_i64 || !starts || !nonmono || !items ||
      !witems || !cpos || !clen || !keys || !gs || !pcnt || !item_off || !n_proc || !n_blend || !scr.widx || !scr.wz ||
      !scr.scan || !scr.torder || !scr.rows || !pbits || !prec)
    return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  // (no splat_off / pos_of: the fused path never maps splats to their list positions)
  ts_impl_bin_count(cap, so.bbox, so.md, tx, ty, cam.near_, cam.far_, w, starts, nullptr, nullptr, nullptr, st, &dyn,
                    so.prect, so.qbits);
  // tile pairs M = starts[T] (and the longest list) recorded; overflow when M > cap_M
  // (and the longest list: the sort kernels launched are those of lists up to cap_L)
  const int64_t capL = ws->capL > 0 ? ws->capL : ((int64_t)1 << 40);
  k_caps_check<<<1, 1, 0, st>>>(starts + T, capM, ovf, need + 1, w.dev_i64 + 1, need + 3, capL, nullptr, nullptr);
  ts_impl_bin_sort(cap, tx, ty, so.md, w, starts, nullptr, capL, keys, gs, items, nullptr, nonmono, st,
                   reinterpret_cast<uint32_t*>(pcnt), &dyn);
  BinsView bv{starts, nullptr, items, nullptr, nonmono, witems, cpos, clen};
  const float* colors = nullptr;
  if (colors_tet && cmap) {
    float* c = ws->colors.get<float>(cap * 3);
    if (!c) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
    k_gather_colors<<<(int)((cap + 255) / 256 < 4096 ? (cap + 255) / 256 : 4096), 256, 0, st>>>(cap, so.tet_ids,
                                                                                                colors_tet, c, nullptr);
    colors = c;
  }
  // window + pair numbering over the M capacity (the M valid positions scanned)
  ts_impl_forward_prepare(tx, ty, bv, capM, so.md, n_w, cam.near_, cam.far_, so.rec, item_off, st, &scr, true, &dyn,
                          starts + T, so.prect);
  k_caps_check<<<1, 1, 0, st>>>(item_off + capM, capP, ovf, need + 2, nullptr, nullptr, 0, need, ws->need_out);
  ts_impl_forward(tx, ty, bv, so.rec, colors,
                  Scene64{nullptr, nullptr, so.f, so.bbox, so.vert_ids, deform, make_grid(R), cam}, cam.width,
                  cam.height, s, t_stop, item_off, capP, pbits, prec, nmap, dmap, omap, colors ? cmap : nullptr,
                  n_proc, n_blend, st, &scr, &dyn);
  ws->K = cap;
  ws->M = capM;
  ws->P = capP;
  ws->maxL = -1;
  ws->tiles_x = tx;
  ws->tiles_y = ty;
  ws->R = R;
  ws->cam = cam;
  ws->s = s;
  ws->color = colors != nullptr;
  ws->valid = true;
  out_counts[0] = out_counts[1] = out_counts[2] = out_counts[3] = -1;  // on the device: ts_view_collect
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ws_fail(TS_ECUDA, cudaGetErrorString(e));
  return TS_OK;
}

int ts_view_forward(ts_workspace* ws, const double* sdf, const double* deform, int32_t R, const ts_camera* camp,
                    double s, const int32_t* active, int64_t n_active, int32_t n_w, double t_stop,
                    const float* colors_tet, float* nmap, float* dmap, float* omap, float* cmap,
                    int64_t* out_counts, void* stream) {
  TS_NVTX("ts_view_forward");
  if (!ws || !sdf || !deform || !camp || R < 1 || n_active < 0 || (n_active > 0 && !active) || !nmap || !dmap ||
      !omap || !out_counts)
    return ws_fail(TS_EINVAL, "ts_view_forward: bad arguments");
  if (n_w < 1) return ws_fail(TS_EINVAL, "resorting window must be >= 1");
  if (camp->width < 1 || camp->height < 1 || camp->width > 32767 || camp->height > 32767)
    return ws_fail(TS_EINVAL, "image size must be in [1, 32767]");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Camera cam = cam_of(camp);
  const int tx = (cam.width + TS_TILE - 1) / TS_TILE, ty = (cam.height + TS_TILE - 1) / TS_TILE;
  const int64_t T = (int64_t)tx * ty, HW = (int64_t)cam.width * cam.height;
  ws->valid = false;
  ws->dyn = ws->capM > 0 && ws->capP > 0;
  if (ws->dyn) return view_forward_dyn(ws, sdf, deform, R, cam, s, active, n_active, n_w, t_stop, colors_tet, nmap,
                                       dmap, omap, cmap, out_counts, st);
  // ---- K2 build_scene ----------------------------------------------------------------------
  const int64_t cap = n_active > 0 ? n_active : 1;
  // no FP64 proj / depths: the forward's exact path re-projects the few splats it needs
  SceneOut so{ws->tet_ids.get<int32_t>(cap), ws->vert_ids.get<int32_t>(cap * 4), nullptr,
              nullptr, ws->f.get<double>(cap * 4), nullptr,
              ws->md.get<double>(cap), nullptr, ws->bbox.get<double>(cap * 4),
              ws->rec.get<SplatRec>(cap), ws->prect.get<int2>(cap)};
  int64_t* scratch = ws->scratch.get<int64_t>(compact_blocks((cap > T ? cap : T) + 1, 1));
  so.qbits = reinterpret_cast<uint32_t*>(ws->qbits.get<unsigned char>(kQBytes));
  if (!so.tet_ids || !so.rec || !scratch || !so.qbits) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  cudaMemsetAsync(so.qbits, 0, kQBytesZero, st);                                          // keys, max md
  cudaMemsetAsync(reinterpret_cast<unsigned char*>(so.qbits) + kQBytesZero, 0xff, kQBytes - kQBytesZero, st);  // min md
  // the scene indexed by active tet (k_cull_emit: no compaction, culled tets keep their slot)
  int64_t* nvis_dev = ws->need.get<int64_t>(4);  // (the sync-free path's counts; free here)
  if (!nvis_dev) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  ts_impl_build_scene_inplace(sdf, deform, R, cam, s, active, n_active, so, nvis_dev, st);
  const int64_t K = n_active > 0 ? n_active : 0;
  // ---- K3-K5 bins ----------------------------------------------------------------------------
  BinWork w;
  w.br = reinterpret_cast<BinRec*>(ws->br.get<int4>(cap));
  w.q = ws->q.get<uint32_t>(cap);
  w.splat_cnt = ws->splat_cnt.get<int32_t>(cap);
  w.tile_cnt = ws->tile_cnt.get<int32_t>(T);
  w.scratch = scratch;
  w.dev_i64 = ws->dev_i64.get<int64_t>(2);
  int64_t* starts = ws->starts.get<int64_t>(T + 1);
  uint8_t* nonmono = ws->nonmono.get<uint8_t>(T);
  if (!w.br || !w.q || !w.splat_cnt || !w.tile_cnt || !w.dev_i64 || !starts || !nonmono)
    return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  int64_t M = 0, maxL = 0;
  ts_impl_bin_count(K, so.bbox, so.md, tx, ty, cam.near_, cam.far_, w, starts, nullptr, &M, &maxL, st, nullptr,
                    so.prect, so.qbits);
  int64_t Kvis = 0;  // reported only; the bin count above already waited for the scene build
  cudaMemcpyAsync(&Kvis, nvis_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st);  // pageable: returns when done
  int32_t* items = ws->items.get<int32_t>(M);
  int32_t* witems = ws->witems.get<int32_t>(M);
  int32_t* cpos = ws->cpos.get<int32_t>(M);
  int32_t* clen = ws->clen.get<int32_t>(T);
  uint64_t* keys = ws->keys.get<uint64_t>(M);
  uint64_t* gs = maxL > 16384 ? ws->gsort.get<uint64_t>(2 * M) : nullptr;
  if (!items || !witems || !cpos || !clen || !keys || (maxL > 16384 && !gs))
    return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  // the sort also writes each position's depth key into the pair-count scratch, which k_window
  // reads (each tile before k_window_counts overwrites it with the tile's pair counts)
  int32_t* pcnt = ws->pcnt.get<int32_t>(M);
  if (!pcnt) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  if (M > 0)
    ts_impl_bin_sort(K, tx, ty, so.md, w, starts, nullptr, maxL, keys, gs, items, nullptr, nonmono, st,
                     reinterpret_cast<uint32_t*>(pcnt));
  else cudaMemsetAsync(nonmono, 0, T, st);
  BinsView bv{starts, nullptr, items, nullptr, nonmono, witems, cpos, clen};
  // ---- colors of the visible splats ------------------------------------------------------
  const float* colors = nullptr;
  if (colors_tet && cmap && K > 0) {
    float* c = ws->colors.get<float>(K * 3);
    if (!c) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
    k_gather_colors<<<(int)((K + 255) / 256 < 4096 ? (K + 255) / 256 : 4096), 256, 0, st>>>(K, so.tet_ids, colors_tet,
                                                                                            c, nullptr);
    colors = c;
  }
  // ---- K6 forward ------------------------------------------------------------------------------
  int32_t* n_proc = ws->n_proc.get<int32_t>(HW);
  int32_t* n_blend = ws->n_blend.get<int32_t>(HW);
  int64_t* item_off = ws->item_off.get<int64_t>(M + 1);
  if (!n_proc || !n_blend || !item_off) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  int64_t P = 0;
  ViewScratch scr;
  scr.widx = ws->widx.get<int32_t>(M);
  scr.wz = ws->wz.get<double>(M);
  scr.cnt = pcnt;
  scr.scan = ws->pscan.get<int64_t>(compact_blocks(M));
  scr.torder = ws->torder.get<int32_t>(T);
  scr.rows = ws->rows.get<float>(24 * (M > K ? M : (K > 0 ? K : 1)));  // kGr floats per splat
  if (!scr.widx || !scr.wz || !scr.cnt || !scr.scan || !scr.torder || !scr.rows)
    return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  if (K > 0 && M > 0)
    P = ts_impl_forward_prepare(tx, ty, bv, M, so.md, n_w, cam.near_, cam.far_, so.rec, item_off, st, &scr, true,
                                nullptr, nullptr, so.prect);
  uint32_t* pbits = ws->pair_bits.get<uint32_t>(TS_PAIR_BIT_WORDS(P));
  float4* prec = ws->pair_rec.get<float4>(P);
  if (!pbits || !prec) return ws_fail(TS_ENOMEM, "ts_view_forward: out of device memory");
  if (K > 0 && M > 0) {
    ts_impl_forward(tx, ty, bv, so.rec, colors, Scene64{nullptr, nullptr, so.f, so.bbox, so.vert_ids, deform, make_grid(R), cam}, cam.width, cam.height, s,
                    t_stop, item_off, P, pbits, prec, nmap, dmap, omap, colors ? cmap : nullptr, n_proc, n_blend,
                    st, &scr);
  } else {
    cudaMemsetAsync(nmap, 0, sizeof(float) * 3 * HW, st);
    cudaMemsetAsync(dmap, 0, sizeof(float) * HW, st);
    cudaMemsetAsync(omap, 0, sizeof(float) * HW, st);
    if (cmap) cudaMemsetAsync(cmap, 0, sizeof(float) * 3 * HW, st);
    cudaMemsetAsync(n_proc, 0, sizeof(int32_t) * HW, st);
    cudaMemsetAsync(n_blend, 0, sizeof(int32_t) * HW, st);
  }
  ws->K = K;
  ws->Kvis = Kvis;
  ws->M = M;
  ws->P = P;
  ws->maxL = maxL;
  ws->tiles_x = tx;
  ws->tiles_y = ty;
  ws->R = R;
  ws->cam = cam;
  ws->s = s;
  ws->color = colors != nullptr;
  ws->valid = true;
  out_counts[0] = Kvis;
  out_counts[1] = M;
  out_counts[2] = P;
  out_counts[3] = maxL;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ws_fail(TS_ECUDA, cudaGetErrorString(e));
  return TS_OK;
}

static int view_backward(ts_workspace* ws, const double* deform, const float* const maps[4],
                         const float* const dmaps[4], float* d_vert, float* d_color, float* status, void* stream,
                         const Fx* fx) {
  if (!ws || !ws->valid) return ws_fail(TS_EINVAL, "ts_view_backward: no forward state in the workspace");
  if (!deform || !maps || !dmaps || !(d_vert || fx) || !maps[0] || !maps[1] || !maps[2] || !dmaps[0] ||
      !dmaps[1] || !dmaps[2])
    return ws_fail(TS_EINVAL, "ts_view_backward: bad arguments");
  if (ws->K == 0 || ws->M == 0) return TS_OK;
  // fixed-point rows are int64: twice the forward's kGr floats per list position (grow-only)
  if (fx && !ws->rows.get<float>(2 * 24 * (size_t)(ws->K > ws->M ? ws->K : ws->M)))
    return ws_fail(TS_ENOMEM, "ts_view_backward_fx: out of device memory");
  Dyn dyn;
  dyn.K = nullptr;  // every scene slot is valid (culled ones skipped by k_chain)
  dyn.ovf = reinterpret_cast<int*>(ws->ovf.p);
  ViewScratch scr;  // sized by the forward of this view
  scr.torder = reinterpret_cast<int32_t*>(ws->torder.p);
  scr.rows = reinterpret_cast<float*>(ws->rows.p);
  const float* m4[4] = {maps[0], maps[1], maps[2], ws->color ? maps[3] : nullptr};
  const float* d4[4] = {dmaps[0], dmaps[1], dmaps[2], ws->color ? dmaps[3] : nullptr};
  BinsView bv{reinterpret_cast<int64_t*>(ws->starts.p), nullptr, reinterpret_cast<int32_t*>(ws->items.p), nullptr,
              reinterpret_cast<uint8_t*>(ws->nonmono.p), reinterpret_cast<int32_t*>(ws->witems.p),
              reinterpret_cast<int32_t*>(ws->cpos.p), reinterpret_cast<int32_t*>(ws->clen.p)};
  ts_impl_backward(ws->tiles_x, ws->tiles_y, bv, ws->M, ws->K, reinterpret_cast<SplatRec*>(ws->rec.p),
                   ws->color ? reinterpret_cast<float*>(ws->colors.p) : nullptr,
                   reinterpret_cast<double*>(ws->f.p), reinterpret_cast<int32_t*>(ws->vert_ids.p),
                   reinterpret_cast<int32_t*>(ws->tet_ids.p), deform, ws->R, ws->cam,
                   reinterpret_cast<int64_t*>(ws->item_off.p), reinterpret_cast<uint32_t*>(ws->pair_bits.p),
                   reinterpret_cast<float4*>(ws->pair_rec.p), m4, d4,
                   reinterpret_cast<int32_t*>(ws->n_proc.p), d_vert, ws->color ? d_color : nullptr,
                   reinterpret_cast<cudaStream_t>(stream), &scr, status, nullptr, 0, nullptr, ws->dyn ? &dyn : nullptr,
                   fx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ws_fail(TS_ECUDA, cudaGetErrorString(e));
  return TS_OK;
}

int ts_view_backward(ts_workspace* ws, const double* deform, const float* const maps[4], const float* const dmaps[4],
                     float* d_vert, float* d_color, float* status, void* stream) {
  TS_NVTX("ts_view_backward");
  if (!d_vert) return ws_fail(TS_EINVAL, "ts_view_backward: bad arguments");
  return view_backward(ws, deform, maps, dmaps, d_vert, d_color, status, stream, nullptr);
}

int ts_view_backward_fx(ts_workspace* ws, const double* deform, const float* const maps[4],
                        const float* const dmaps[4], int64_t* d_vert_fx, int64_t* d_color_fx, float* status,
                        void* stream) {
  TS_NVTX("ts_view_backward_fx");
  if (!ws || !d_vert_fx) return ws_fail(TS_EINVAL, "ts_view_backward_fx: bad arguments");
  const int64_t n = (int64_t)ws->R + 1;
  Fx fx;
  fx.vert = reinterpret_cast<long long*>(d_vert_fx);
  fx.color = reinterpret_cast<long long*>(d_color_fx);
  fx.bad = reinterpret_cast<unsigned long long*>(d_vert_fx + 4 * n * n * n);
  return view_backward(ws, deform, maps, dmaps, nullptr, nullptr, status, stream, &fx);
}

// n_blend of the last forward (H*W int32, device) — for parity checks
const int32_t* ts_view_n_blend(ts_workspace* ws) { return ws ? reinterpret_cast<int32_t*>(ws->n_blend.p) : nullptr; }

}  // extern "C"
