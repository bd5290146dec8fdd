// scene.cu — K1 prefilter + compaction and K2 projection / splat setup.
//
// K1 replaces splat.prefilter (splat.py:66-69 -> alpha_max splat.py:42-55): one FP64
//    alpha_max per tet of the implicit Kuhn grid, survivors emitted in increasing id.
// K2 replaces splat.build_scene (splat.py:203-245): projection (camera.py:56-67), the
//    frustum/image cull (splat.py:216-221), the in-tet gradient normal (field.py:140-177,
//    cross-product form of _core.pyx:474-514), mean depth, bbox, alpha_max, and the
//    compact FP32 compositing record — all fused into one order-preserving compaction.
// Both are HBM-bound gathers: each thread owns one tet, vertex data is reused via L1/L2.
#include "internal.cuh"
#include "scan.cuh"

namespace ts {

// alpha_max >= threshold (splat.py:42-55), FP64 with numpy's operation order
__device__ __forceinline__ bool alpha_max_pass(const double f[4], double s, double thr, double* amax_out) {
  double fmx = f[0], fmn = f[0];
  for (int i = 1; i < 4; ++i) {
    fmx = f[i] > fmx ? f[i] : fmx;
    fmn = f[i] < fmn ? f[i] : fmn;
  }
  double a = dmul(s, fmx), b = dmul(s, fmn);
  double ratio = exp(dsub(softplus_d(-a), softplus_d(-b)));
  double am = dsub(1.0, ratio);
  am = am > 0.0 ? am : 0.0;
  if (amax_out) *amax_out = am;
  return am >= thr;
}

// alpha_max >= thr for a tet with corner SDF values f: alpha_max = sigmoid(-b) (1 - e^{-(a-b)}),
// a = s fmax >= b = s fmin, estimated in FP32 from the FP64 difference (relative error ~1e-6);
// the reference's FP64 evaluation errs by < 1e-13 absolute, so outside a 2e-6 relative band
// around the threshold the decision is certain and only the tets inside it take the FP64
// softplus path
__device__ __forceinline__ bool prefilter_pass(const double f[4], double s, double thr) {
  double fmx = f[0], fmn = f[0];
  for (int i = 1; i < 4; ++i) {
    fmx = f[i] > fmx ? f[i] : fmx;
    fmn = f[i] < fmn ? f[i] : fmn;
  }
  const double a = dmul(s, fmx), b = dmul(s, fmn);
  const float y = (float)(-b), d = (float)dsub(a, b);
  const float ey = expf(-fabsf(y)), r = 1.0f / (1.0f + ey);
  const float sig = y >= 0.f ? r : ey * r;
  const float est = sig * -expm1f(-d);
  const float tf = (float)thr;
  if (fabsf(est - tf) > 2e-6f * tf + 1e-12f) return est > tf;
  return alpha_max_pass(f, s, thr, nullptr);
}

// K1 per cell: the 8 corner samples of a cell are loaded once for its 6 tets (tet id = cell * 6
// + p, cells z-fastest = tet-id order), two consecutive cells per thread; survivors compacted
// in increasing id with a decoupled look-back (single pass).
constexpr int kPfCells = 2;
__global__ void __launch_bounds__(256) k_prefilter_cells(int64_t C, Grid G, const double* __restrict__ sdf, double s,
                                                         double thr, int32_t* __restrict__ out,
                                                         unsigned long long* __restrict__ status,
                                                         unsigned long long* __restrict__ ticket, int64_t nb) {
  __shared__ int wcnt[8];
  __shared__ long long pre_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tile = lb_tile(ticket);
  const int64_t c0 = (int64_t)tile * (256 * kPfCells) + (int64_t)threadIdx.x * kPfCells;
  uint32_t mask = 0;  // bit k * 6 + p: tet p of cell c0 + k passes
#pragma unroll
  for (int k = 0; k < kPfCells; ++k) {
    const int64_t c = c0 + k;
    if (c >= C) break;
    const uint32_t q = G.dR.div((uint32_t)c);  // ix*R + iy
    const uint32_t iz = (uint32_t)c - q * (uint32_t)G.R;
    const uint32_t ix = G.dR.div(q);
    const uint32_t iy = q - ix * (uint32_t)G.R;
    const uint32_t n = (uint32_t)G.n, v0 = ix + n * (iy + n * iz);
    double fc[8];
#pragma unroll
    for (int lc = 0; lc < 8; ++lc) fc[lc] = __ldg(sdf + v0 + (lc & 1) + n * (((lc >> 1) & 1) + n * ((lc >> 2) & 1)));
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const double f[4] = {fc[perm_corner(p, 0)], fc[perm_corner(p, 1)], fc[perm_corner(p, 2)], fc[perm_corner(p, 3)]};
      if (prefilter_pass(f, s, thr)) mask |= 1u << (k * 6 + p);
    }
  }
  const int cnt = __popc(mask);
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wcnt[wid] = v;
  __syncthreads();
  int before = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    before += (w < wid) ? wcnt[w] : 0;
    agg += wcnt[w];
  }
  if (wid == 0) {
    const long long pr = lb_exclusive(status, tile, agg);
    if (lane == 0) pre_s = pr;
  }
  __syncthreads();
  long long pos = pre_s + before + v - cnt;
  for (uint32_t m = mask; m; m &= m - 1u) {
    const int b = __ffs(m) - 1;
    out[pos++] = (int32_t)((c0 + b / 6) * 6 + b % 6);
  }
  if (tile == nb - 1 && threadIdx.x == 0) *reinterpret_cast<long long*>(ticket) = pre_s + agg;
}

struct CullF {
  const int32_t* active;
  const double* sdf;
  const double* deform;
  Grid G;
  Camera cam;
  double s;
  SceneOut out;

  __device__ void project4(int64_t i, uint32_t v[4], double P[4][3], double px[4], double py[4],
                           double z[4]) const {
    int xyz[4][3];
    tet_corners((uint32_t)active[i], G, xyz, v);
    for (int c = 0; c < 4; ++c) {
      double pc[3];
      vertex_pos_xyz(xyz[c], v[c], G, deform, P[c]);
      project_point(cam, P[c], px[c], py[c], z[c], pc);
    }
  }
  __device__ static void bounds(const double px[4], const double py[4], const double z[4], double& dmin,
                                double& xmin, double& xmax, double& ymin, double& ymax) {
    dmin = z[0]; xmin = xmax = px[0]; ymin = ymax = py[0];
    for (int c = 1; c < 4; ++c) {
      dmin = z[c] < dmin ? z[c] : dmin;
      xmin = px[c] < xmin ? px[c] : xmin;
      xmax = px[c] > xmax ? px[c] : xmax;
      ymin = py[c] < ymin ? py[c] : ymin;
      ymax = py[c] > ymax ? py[c] : ymax;
    }
  }
  // projected tet, kept between the visibility test and the emission (k_compact_lb); the
  // positions are re-formed at emission (an L1 hit) instead of living across the look-back
  struct State {
    uint32_t v[4];
    double px[4], py[4], z[4];
  };
  __device__ bool visible(const double px[4], const double py[4], const double z[4]) const {
    double dmin, xmin, xmax, ymin, ymax;
    bounds(px, py, z, dmin, xmin, xmax, ymin, ymax);
    return (dmin > cam.near_) && (dmin <= cam.far_) && (xmax >= 0.0) && (xmin <= (double)cam.width) &&
           (ymax >= 0.0) && (ymin <= (double)cam.height);
  }
  __device__ bool pred(int64_t i) const {
    State st;
    return pred(i, st);
  }
  __device__ bool pred(int64_t i, State& st) const {
    double P[4][3];
    project4(i, st.v, P, st.px, st.py, st.z);
    return visible(st.px, st.py, st.z);
  }
  // fused view path: an active tet this view culls keeps its slot (records.cuh kCulledRect)
  __device__ void cull(int64_t i) const {
    out.tet_ids[i] = active[i];
    out.prect[i] = make_int2(kCulledRect, kCulledRect);
    *reinterpret_cast<int2*>(out.rec + i) = make_int2(kCulledRect, kCulledRect);
  }
  __device__ void emit(int64_t i, int64_t k, const State& st) const {
    const uint32_t* v = st.v;
    double P[4][3];
    {
      int xyz[4][3];
      uint32_t vv[4];
      tet_corners((uint32_t)active[i], G, xyz, vv);
      for (int c = 0; c < 4; ++c) vertex_pos_xyz(xyz[c], vv[c], G, deform, P[c]);
    }
    const double *px = st.px, *py = st.py, *z = st.z;
    double dmin, xmin, xmax, ymin, ymax;
    bounds(px, py, z, dmin, xmin, xmax, ymin, ymax);
    double f[4], proj[8], bb[4] = {xmin, ymin, xmax, ymax};
    for (int c = 0; c < 4; ++c) {
      f[c] = __ldg(sdf + v[c]);
      proj[2 * c] = px[c];
      proj[2 * c + 1] = py[c];
    }
    // 16-byte stores (the arrays are 16-byte aligned per splat)
    reinterpret_cast<int4*>(out.vert_ids)[k] = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
    if (out.proj) {  // optional: the fused view path re-projects in its exact path instead
      double2* pj = reinterpret_cast<double2*>(out.proj + k * 8);
      for (int c = 0; c < 4; ++c) pj[c] = make_double2(px[c], py[c]);
      double2* dz = reinterpret_cast<double2*>(out.depths + k * 4);
      dz[0] = make_double2(z[0], z[1]);
      dz[1] = make_double2(z[2], z[3]);
    }
    double2* ff = reinterpret_cast<double2*>(out.f + k * 4);
    double2* bx = reinterpret_cast<double2*>(out.bbox + k * 4);
    ff[0] = make_double2(f[0], f[1]);
    ff[1] = make_double2(f[2], f[3]);
    bx[0] = make_double2(bb[0], bb[1]);
    bx[1] = make_double2(bb[2], bb[3]);
    out.tet_ids[k] = active[i];
    double g[3], c1[3], c2[3], c3[3], nrm[3] = {0.0, 0.0, 0.0};
    tet_gradient(P, f, g, c1, c2, c3);
    double gn = sqrt(dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2])));
    if (gn >= 1e-8)
      for (int c = 0; c < 3; ++c) nrm[c] = ddiv(g[c], gn);
    if (out.normals)  // optional FP64 outputs (the fused view pipeline needs neither)
      for (int c = 0; c < 3; ++c) out.normals[k * 3 + c] = nrm[c];
    double md = dmul(dadd(dadd(dadd(z[0], z[1]), z[2]), z[3]), 0.25);  // == the division by 4, exactly
    out.md[k] = md;
    if (out.amax) {
      double am;
      alpha_max_pass(f, s, 0.0, &am);
      out.amax[k] = am;
    }
    // never-blend certificate (records.cuh): A_i = grad f . (P_i - o) / z_i, o the camera centre
    double amin = 1e300;
    for (int c = 0; c < 4; ++c) {
      double a = 0.0;
      for (int q = 0; q < 3; ++q)
        a += g[q] * (P[c][q] + (cam.R[q] * cam.t[0] + cam.R[3 + q] * cam.t[1] + cam.R[6 + q] * cam.t[2]));
      amin = fmin(amin, a / z[c]);
    }
    const double gn2 = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    const SplatRec r = make_record(proj, z, f, nrm, md, bb, cam.width, cam.height,
                                   out.certify && amin > 1e-9 * gn2 ? amin : 0.0);
    out.rec[k] = r;
    if (out.prect) out.prect[k] = make_int2(r.rx, r.ry);
    if (out.qbits) {  // (fused path) the drop tables of records.cuh
      const uint32_t q = depth_key(md, cam.near_, cam.far_);
      if (!rect_empty(make_int2(r.rx, r.ry))) {
        const uint32_t h = qhash(q);
        atomicOr(out.qbits + (h >> 5), 1u << (h & 31));
      }
      unsigned long long* mx = qtab_max(out.qbits);
      const unsigned long long bits = (unsigned long long)__double_as_longlong(md), h2 = qhash2(q);
      atomicMax(mx + h2, bits);
      atomicMin(mx + kQTab + h2, bits);
    }
  }
};

// Record preparation for a scene that arrived as FP64 arrays (e.g. uploaded).
__global__ void k_prepare_records(int64_t K, const double* __restrict__ proj, const double* __restrict__ depths,
                                  const double* __restrict__ f, const double* __restrict__ normals,
                                  const double* __restrict__ md, const double* __restrict__ bbox, int width,
                                  int height, SplatRec* __restrict__ rec, bool certify) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    double p[8], z[4], ff[4], n[3], b[4];
    for (int i = 0; i < 8; ++i) p[i] = proj[k * 8 + i];
    for (int i = 0; i < 4; ++i) { z[i] = depths[k * 4 + i]; ff[i] = f[k * 4 + i]; b[i] = bbox[k * 4 + i]; }
    for (int i = 0; i < 3; ++i) n[i] = normals[k * 3 + i];
    rec[k] = make_record(p, z, ff, n, md[k], b, width, height, certify ? backfacing_amin(p, z, ff) : 0.0);
  }
}

// Fused view path: the scene indexed by active tet (its scene is internal, so no compaction:
// no look-back, one projection per tet); culled tets get the kCulledRect sentinel, which
// k_bin_count and k_chain skip.  n_vis receives the visible count (reported only).
#ifndef TS_CULL_MINB
#define TS_CULL_MINB 1
#endif
__global__ void __launch_bounds__(256, TS_CULL_MINB) k_cull_emit(int64_t n, CullF f, unsigned long long* __restrict__ n_vis) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool vis = false;
    if (i < n) {
      CullF::State st;
      vis = f.pred(i, st);
      if (vis) f.emit(i, i, st);
      else f.cull(i);
    }
    const unsigned m = __ballot_sync(0xffffffffu, vis);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(n_vis, (unsigned long long)__popc(m));
  }
}

__global__ void k_cull_slot0(SceneOut out) {
  out.tet_ids[0] = 0;
  out.prect[0] = make_int2(kCulledRect, kCulledRect);
  *reinterpret_cast<int2*>(out.rec) = make_int2(kCulledRect, kCulledRect);
}

}  // namespace ts

using namespace ts;

void ts_impl_build_scene_inplace(const double* sdf, const double* deform, int R, const Camera& cam, double s,
                                 const int32_t* active, int64_t n_active, const SceneOut& out, int64_t* n_vis,
                                 cudaStream_t st) {
  cudaMemsetAsync(n_vis, 0, sizeof(int64_t), st);
  if (n_active <= 0) {  // the one capacity slot holds no splat
    k_cull_slot0<<<1, 1, 0, st>>>(out);
    return;
  }
  CullF f{active, sdf, deform, make_grid(R), cam, s, out};
  f.out.certify = !(ts_impl_debug_flags() & 128);
  int blocks = (int)((n_active + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_cull_emit<<<blocks, 256, 0, st>>>(n_active, f, reinterpret_cast<unsigned long long*>(n_vis));
}

// host entry points used by abi.cu
int64_t ts_impl_prefilter(const double* sdf, int R, double s, double thr, int32_t* out_active,
                          int64_t* scratch, cudaStream_t st) {
  // scratch: compact_blocks(6 R^3) >= nb + 1 entries (a tile = 512 cells = 3072 tets)
  const int64_t C = (int64_t)R * R * R;
  const int64_t nb = (C + 256 * kPfCells - 1) / (256 * kPfCells);
  cudaMemsetAsync(scratch, 0, sizeof(int64_t) * (nb + 1), st);
  k_prefilter_cells<<<(unsigned)nb, 256, 0, st>>>(C, make_grid(R), sdf, s, thr, out_active,
                                                  reinterpret_cast<unsigned long long*>(scratch),
                                                  reinterpret_cast<unsigned long long*>(scratch + nb), nb);
  int64_t h = 0;
  cudaMemcpyAsync(&h, scratch + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}

int64_t ts_impl_build_scene(const double* sdf, const double* deform, int R, const Camera& cam, double s,
                            const int32_t* active, int64_t n_active, const SceneOut& out, int64_t* scratch,
                            cudaStream_t st) {
  CullF f{active, sdf, deform, make_grid(R), cam, s, out};
  f.out.certify = !(ts_impl_debug_flags() & 128);
  int64_t* d_total = compact_state<CullF>(n_active, f, scratch, st);  // scratch: compact_blocks(n, 1)
  int64_t h = 0;
  cudaMemcpyAsync(&h, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}


void ts_impl_prepare_records(int64_t K, const double* proj, const double* depths, const double* f,
                             const double* normals, const double* md, const double* bbox, int width, int height,
                             SplatRec* rec, cudaStream_t st) {
  if (K <= 0) return;
  int blocks = (int)((K + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prepare_records<<<blocks, 256, 0, st>>>(K, proj, depths, f, normals, md, bbox, width, height, rec,
                                            !(ts_impl_debug_flags() & 128));
}
