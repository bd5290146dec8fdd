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

// Build the compact record from the FP64 scene values of one splat.
__device__ inline SplatRec make_record(const double proj[8], const double depths[4], const double f[4],
                                       const double normal[3], double md, const double bbox[4],
                                       int width, int height) {
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
