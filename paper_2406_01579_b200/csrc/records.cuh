// records.cuh — splat records shared by the binning, compositing and gradient kernels.
//
// A visible splat exists in two forms:
//  * the FP64 SplatScene arrays of the reference (splat.py:177-200: proj, depths, f,
//    normals, mean_depth, alpha_max, bbox), kept for the exact paths (tile keys, exact
//    hit fallback) and the public API;
//  * a compact 96-byte FP32 SplatRec that the compositing kernels stage through shared
//    memory.  Its pixel rectangle is the reference's inclusive bbox test (_core.pyx:80)
//    turned into integer pixel bounds computed exactly in FP64, and its vertex
//    coordinates are anchored at the rectangle's first pixel so FP32 keeps ~1e-6 px.
#pragma once
#include "common.cuh"

namespace ts {

constexpr double kEpsDet = 2e-12;         // _core.pyx:12
constexpr float kBandScale = 1.220703125e-4f;  // 2^-13: edge-function ambiguity band / M^2

struct __align__(16) SplatRec {
  int32_t rx;       // ix0 | ix1 << 16  (int16 each; empty when ix0 > ix1)
  int32_t ry;       // iy0 | iy1 << 16
  float band;       // |edge function| below this -> exact FP64 fallback
  uint32_t flags;   // bits 0-3: face f valid (|det64| >= 2e-12); bit 4: always use fallback
  float vx[4], vy[4];  // projected vertices minus (ix0, iy0)
  float z[4];          // camera-space depths
  float f[4];          // SDF samples as f0, f1-f0, f2-f0, f3-f0 (deltas keep FP32 error ~ spread)
  float n[3];          // unit normal (zero when undefined)
  float md;            // mean depth
};
static_assert(sizeof(SplatRec) == 96, "SplatRec must be 96 bytes");

// local vertex triples of the four faces (_core.pyx:14-18, splat.py:19)
__host__ __device__ constexpr int face_vert(int fi, int j) {
  return (fi == 0) ? (j + 1) : (j < fi ? j : j + 1);
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Never-blend certificate ("back-facing splats").  The SDF is linear over the
// tet: along the ray of pixel p (direction d_p scaled to unit depth from the camera centre o)
// the SDF at depth z is f = A(p) z + f_lin(o) with A(p) = grad f . d_p affine in p, so
// f_next - f_prev = A(p) (z_out - z_in).  When A > 0 at the four projected vertices
// (A_i = grad f . (P_i - o) / z_i, hence over the whole hull) no ray through the tet sees the
// SDF decrease, so the reference's alpha = 1 - exp(sp(-s f_prev) - sp(-s f_next)) is <= 0 —
// up to its FP64 rounding, which can only matter where f_next - f_prev is tiny, i.e. near
// the line of the edge e shared by the entry and exit faces F, B: with the w = 1/z planes
// w_F, w_B of those faces, z_out - z_in = (w_F - w_B)(p) / (w_in w_out)
// >= z_min^2 kappa_e dist(p, line e), kappa_e = |grad(w_F - w_B)| (w_F - w_B vanishes on e),
// so f_next - f_prev >= A_min z_min^2 kappa_e dist(p, line e).  The certificate asks that no
// pixel centre of the rectangle lies within r_e of any edge line, r_e covering the FP64 error
// of the reference's f_prev - f_next (~1e-15 (1 + C M / |det|) max|f|, C the coordinate
// magnitude, M the splat extent) and of its face-containment test (~1e-15 C M / |e|), both
// taken 10^6 times larger, plus the FP32 error of this evaluation on the record's anchored
// geometry (1e-4 px; gradients within 2%, enforced).  Then every pixel either misses the
// hull (no two hits) or lies inside it away from all edges (exactly F and B hit,
// f_next - f_prev > the error): no pixel of the splat blends in the reference, for any
// steepness.  Its rectangle is emptied; the binning keeps the FP64 bbox, so tile lists, the
// window and n_proc are unchanged.  About half of the splats of a closed surface face away
// from the camera (tests/test_gpu_certificate.py: the certified set against the reference's
// blends with early stop disabled).
__device__ __forceinline__ float rcp_approx(float x) {  // <= 1 ulp (the certificate's margins budget for it)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ inline bool never_blends(const SplatRec& r, int nxr, int nyr, double amin, double C, double M,
                                    double fabsmax, double fmx) {
  // one exit, no early returns: lanes leave each edge's scan loop together (a divergent exit
  // inside the unrolled edges kept warps at ~2 active lanes)
  bool ok = nxr <= 64 && nyr <= 64;
  float w[4], zmin = r.z[0], wmax = 0.f;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    ok &= r.z[v] > 0.f;
    w[v] = rcp_approx(r.z[v]);
    zmin = fminf(zmin, r.z[v]);
    wmax = fmaxf(wmax, w[v]);
  }
  float len[6], ilen[6], lmax = 0.f;
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const int va = e < 3 ? 0 : (e < 5 ? 1 : 2), vb = e < 3 ? e + 1 : (e < 5 ? e - 1 : 3);
    const float dx = r.vx[vb] - r.vx[va], dy = r.vy[vb] - r.vy[va], d2 = dx * dx + dy * dy;
    ilen[e] = rsqrt_approx(d2);
    len[e] = d2 * ilen[e];
    lmax = fmaxf(lmax, len[e]);
  }
  // 1/z plane gradients of the faces (pixel units) and their FP32 error bounds
  float gx[4], gy[4], adet[4], gerr[4];
#pragma unroll
  for (int fi = 0; fi < 4; ++fi) {
    const int ia = face_vert(fi, 0), ib = face_vert(fi, 1), ic = face_vert(fi, 2);
    const float m00 = r.vx[ib] - r.vx[ia], m10 = r.vy[ib] - r.vy[ia];
    const float m01 = r.vx[ic] - r.vx[ia], m11 = r.vy[ic] - r.vy[ia];
    const float det = m00 * m11 - m01 * m10;
    ok &= fabsf(det) > 1e-3f * lmax * lmax;  // thin face: not certified
    const float inv = rcp_approx(det), d1 = w[ib] - w[ia], d2 = w[ic] - w[ia];
    gx[fi] = (d1 * m11 - m10 * d2) * inv;
    gy[fi] = (m00 * d2 - m01 * d1) * inv;
    adet[fi] = fabsf(det);
    const float g2 = gx[fi] * gx[fi] + gy[fi] * gy[fi];
    gerr[fi] = (5e-7f * wmax + 1e-5f * g2 * rsqrt_approx(g2)) * 2.f * lmax * fabsf(inv);
  }
  const float am = (float)amin, e64c = (float)(1e-9 * fabsmax), e64f = (float)(1e-9 * fmx);
  const float cm = (float)(C * M);
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const int va = e < 3 ? 0 : (e < 5 ? 1 : 2), vb = e < 3 ? e + 1 : (e < 5 ? e - 1 : 3);
    // the two faces through edge (va, vb) omit the two other vertices
    const int fa = (va != 0 && vb != 0) ? 0 : ((va != 1 && vb != 1) ? 1 : 2);
    const int fb = 6 - va - vb - fa;
    const float kx = gx[fa] - gx[fb], ky = gy[fa] - gy[fb], k2 = kx * kx + ky * ky;
    const float kappa = k2 * rsqrt_approx(k2);
    ok &= kappa > 50.f * (gerr[fa] + gerr[fb]);
    const float dx = r.vx[vb] - r.vx[va], dy = r.vy[vb] - r.vy[va];
    const float e64 = e64c * (1.0f + cm * rcp_approx(fminf(adet[fa], adet[fb]))) + e64f;
    const float rad = fmaxf(2.f * e64 * rcp_approx(am * zmin * zmin * kappa), 1e-9f * cm * ilen[e]) + 1e-4f;
    ok &= rad < 0.25f;  // (false on NaN)
    // distance to the line = |dy (px - xa) - dx (py - ya)| / len: scanned by rows when the line
    // is steeper than 45 degrees (|dy| >= |dx|), else by columns
    const bool by_rows = fabsf(dy) >= fabsf(dx);
    const int n_scan = ok ? (by_rows ? nyr : nxr) : 0;
    const float n_across = (float)((by_rows ? nxr : nyr) - 1);
    const float iu = rcp_approx(by_rows ? dy : dx), slope = (by_rows ? dx : dy) * iu;
    const float ua = by_rows ? r.vx[va] : r.vy[va], wa = by_rows ? r.vy[va] : r.vx[va];
    const float half = rad * len[e] * fabsf(iu) * 1.001f + 1e-6f;  // < 0.36: one candidate per row
    // the line crosses row / column i at c(i) = c0 + slope i; pixel centres sit at j + 0.5, and
    // only the nearest one can be within half of it
    const float c0 = ua + slope * (0.5f - wa) - 0.5f;
    bool near = false;
#pragma unroll 2
    for (int i = 0; i < n_scan; ++i) {
      const float d = fmaf(slope, (float)i, c0);
      const float j = rintf(d);
      near |= fabsf(d - j) <= half && j >= 0.f && j <= n_across;
    }
    ok &= !near;
  }
  return ok;
}

// A_min of the certificate from the projected vertices alone (scene_from_arrays): the SDF is
// linear in Q = z (x, y, 1), a linear image of camera space, f = h.Q + f_lin(o), and
// A_i = h.Q_i / z_i.  Returns 0 when the tet is not robustly back-facing.
__device__ inline double backfacing_amin(const double proj[8], const double z[4], const double f[4]) {
  double Q[4][3], a[3][3], b[3];
  for (int v = 0; v < 4; ++v) {
    Q[v][0] = z[v] * proj[2 * v];
    Q[v][1] = z[v] * proj[2 * v + 1];
    Q[v][2] = z[v];
  }
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) a[i][j] = Q[i + 1][j] - Q[0][j];
    b[i] = f[i + 1] - f[0];
  }
  const double c0 = a[1][1] * a[2][2] - a[1][2] * a[2][1], c1 = a[1][2] * a[2][0] - a[1][0] * a[2][2],
               c2 = a[1][0] * a[2][1] - a[1][1] * a[2][0];
  const double D = a[0][0] * c0 + a[0][1] * c1 + a[0][2] * c2;
  double nrm = 1.0;
  for (int i = 0; i < 3; ++i) nrm *= sqrt(a[i][0] * a[i][0] + a[i][1] * a[i][1] + a[i][2] * a[i][2]);
  if (!(fabs(D) > 1e-9 * nrm)) return 0.0;
  double h[3];
  for (int c = 0; c < 3; ++c) {
    double m[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) m[i][j] = j == c ? b[i] : a[i][j];
    h[c] = (m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
            m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0])) / D;
  }
  double amin = 1e300, hn = sqrt(h[0] * h[0] + h[1] * h[1] + h[2] * h[2]);
  for (int v = 0; v < 4; ++v) amin = fmin(amin, (h[0] * Q[v][0] + h[1] * Q[v][1] + h[2] * Q[v][2]) / z[v]);
  return amin > 1e-9 * hn ? amin : 0.0;
}

// 32-bit depth key of a mean depth (raster.py:132-134, FP64, numpy order)
__device__ __forceinline__ uint32_t depth_key(double md, double near_, double far_) {
  double qq = ddiv(dsub(md, near_), dsub(far_, near_));
  qq = qq < 0.0 ? 0.0 : qq;
  qq = qq > 1.0 ? 1.0 : qq;
  return (uint32_t)(unsigned long long)dmul(qq, 4294967295.0);
}

// Splats left out of the fused view path's tile lists.  A splat whose pixel rectangle is empty
// (certified never to blend, or no pixel centre inside its bbox) is never composited, so the
// only effect of its list entries is on the N_w window of its tile.  The window acts on each
// run of equal depth key independently (a key change is a clean boundary: composite.cu
// window_tile), and inside a run whose members all have the same mean depth it pops in list
// order (ties go to the earlier position).  So removing such a splat leaves the pop order of
// every other entry unchanged when (a) no splat with a non-empty rectangle has its depth key,
// or (b) every splat with its depth key has the same mean depth (lattice-aligned views tie
// thousands of splats per key).  The fused path tests both with hashed tables filled by the
// scene build — a bitmap of the keys of splats with pixels, and per key bucket the min / max
// mean-depth bit pattern (md > 0, so the bits order like the values); hash collisions only
// keep a splat.  List positions (n_proc) are internal to that path.
constexpr int kQHashBits = 24;
constexpr int kQBitWords = 1 << (kQHashBits - 5);
constexpr int kQTabBits = 20;  // mean-depth range buckets
constexpr int kQTab = 1 << kQTabBits;
// one buffer: [kQBitWords] u32 key bitmap | [kQTab] u64 max md bits | [kQTab] u64 min md bits
constexpr size_t kQBytesZero = sizeof(uint32_t) * kQBitWords + sizeof(unsigned long long) * kQTab;
constexpr size_t kQBytes = kQBytesZero + sizeof(unsigned long long) * kQTab;  // the min table starts at ~0
__device__ __forceinline__ uint32_t qhash(uint32_t q) { return (q * 0x9E3779B1u) >> (32 - kQHashBits); }
__device__ __forceinline__ uint32_t qhash2(uint32_t q) { return (q * 0x9E3779B1u) >> (32 - kQTabBits); }
__device__ __forceinline__ unsigned long long* qtab_max(uint32_t* qbits) {
  return reinterpret_cast<unsigned long long*>(qbits + kQBitWords);
}
__device__ __forceinline__ const unsigned long long* qtab_max(const uint32_t* qbits) {
  return reinterpret_cast<const unsigned long long*>(qbits + kQBitWords);
}
// fused view path: the packed rectangle of an active tet the view culls (no splat; the scene
// is indexed by active tet there, composite.cu never sees it) — distinct from every empty
// rectangle a record can carry
constexpr int kCulledRect = INT32_MIN;
__device__ __forceinline__ bool rect_empty(int2 pr) {
  return (int)(short)(pr.x & 0xffff) > (pr.x >> 16) || (int)(short)(pr.y & 0xffff) > (pr.y >> 16);
}

// Build the compact record from the FP64 scene values of one splat.
__device__ inline SplatRec make_record(const double proj[8], const double depths[4], const double f[4],
                                       const double normal[3], double md, const double bbox[4],
                                       int width, int height, double amin = 0.0) {
  SplatRec r;
  // pixel centres xi + 0.5 inside [xmin, xmax] (inclusive, _core.pyx:80): exact in FP64
  double fx0 = ceil(dsub(bbox[0], 0.5)), fx1 = floor(dsub(bbox[2], 0.5));
  double fy0 = ceil(dsub(bbox[1], 0.5)), fy1 = floor(dsub(bbox[3], 0.5));
  // clip to the image (pixels outside are never shaded)
  fx0 = fmax(fx0, 0.0); fy0 = fmax(fy0, 0.0);
  fx1 = fmin(fx1, (double)(width - 1)); fy1 = fmin(fy1, (double)(height - 1));
  int ix0, ix1, iy0, iy1;
  if (!(fx0 <= fx1) || !(fy0 <= fy1)) {  // empty (also catches NaN)
    ix0 = 1; ix1 = 0; iy0 = 1; iy1 = 0;
  } else {
    ix0 = (int)fx0; ix1 = (int)fx1; iy0 = (int)fy0; iy1 = (int)fy1;
  }
  r.rx = (ix0 & 0xffff) | (ix1 << 16);
  r.ry = (iy0 & 0xffff) | (iy1 << 16);
  double M = 1.0 + fmax((double)(ix1 - ix0), (double)(iy1 - iy0));
  for (int v = 0; v < 4; ++v) {
    double ax = dsub(proj[2 * v], (double)ix0), ay = dsub(proj[2 * v + 1], (double)iy0);
    r.vx[v] = (float)ax;
    r.vy[v] = (float)ay;
    M = fmax(M, fmax(fabs(ax), fabs(ay)));
    r.z[v] = (float)depths[v];
    r.f[v] = v == 0 ? (float)f[0] : (float)dsub(f[v], f[0]);  // f0, then exact-ish deltas
  }
  uint32_t flags = 0;
  for (int fi = 0; fi < 4; ++fi) {
    const int ia = face_vert(fi, 0), ib = face_vert(fi, 1), ic = face_vert(fi, 2);
    // identical operation order to _core.pyx:43-49
    double ax = proj[2 * ia], ay = proj[2 * ia + 1];
    double m00 = dsub(proj[2 * ib], ax), m10 = dsub(proj[2 * ib + 1], ay);
    double m01 = dsub(proj[2 * ic], ax), m11 = dsub(proj[2 * ic + 1], ay);
    double det = dsub(dmul(m00, m11), dmul(m01, m10));
    if (!(fabs(det) < kEpsDet)) flags |= 1u << fi;
  }
  float band = (float)(M * M) * kBandScale;
  r.band = band;
  r.flags = flags;
  // faces whose FP32 determinant sign is not certain: always take the exact path
  for (int fi = 0; fi < 4; ++fi) {
    if (!(flags & (1u << fi))) continue;
    const int ia = face_vert(fi, 0), ib = face_vert(fi, 1), ic = face_vert(fi, 2);
    float m00 = r.vx[ib] - r.vx[ia], m10 = r.vy[ib] - r.vy[ia];
    float m01 = r.vx[ic] - r.vx[ia], m11 = r.vy[ic] - r.vy[ia];
    float det = m00 * m11 - m01 * m10;
    if (!(fabsf(det) > band)) r.flags |= 16u;
  }
  r.n[0] = (float)normal[0];
  r.n[1] = (float)normal[1];
  r.n[2] = (float)normal[2];
  r.md = (float)md;
#ifndef TS_NO_NEVER_BLEND
  // certified never to blend (amin > 0: the caller found the tet back-facing): empty
  // rectangle with the anchor kept, bit 5
  if (amin > 0.0 && (r.flags & 31u) == 15u && ix0 <= ix1 && iy0 <= iy1) {
    double C = 0.0, fabsmax = 0.0;
    for (int v = 0; v < 4; ++v) {
      C = fmax(C, fmax(fabs(proj[2 * v]), fabs(proj[2 * v + 1])));
      fabsmax = fmax(fabsmax, fabs(f[v]));
    }
    const double fmx = fmax(fabs(f[1] - f[0]), fmax(fabs(f[2] - f[0]), fabs(f[3] - f[0])));
    if (never_blends(r, ix1 - ix0 + 1, iy1 - iy0 + 1, amin, C + M, M, fabsmax, fmx)) {
      r.rx = (int32_t)((uint32_t)(ix0 & 0xffff) | ((uint32_t)(ix0 - 1) << 16));
      r.flags |= 32u;
    }
  }
#endif
  return r;
}

// FP64 view of the scene for the exact fallback and the chain kernel
struct Scene64 {
  const double* proj;     // [K,4,2]  (nullptr: re-projected from the vertices, see below)
  const double* depths;   // [K,4]    (nullptr with proj)
  const double* f;        // [K,4]
  const double* bbox;     // [K,4]
  // the fused view path stores no proj / depths (96 B per splat of write traffic): the exact
  // path re-projects the splat's vertices with the same FP64 functions (bit-identical values)
  const int32_t* vert_ids;  // [K,4]
  const double* deform;
  Grid G;
  Camera cam;
};

}  // namespace ts
