// common.cuh — shared device helpers for the B200 tetrahedron rasterizer (sm_100a).
//
// Conventions
//  * Geometry that feeds bit-exact decisions (tile rects, depth keys, pixel rects,
//    degenerate-face tests, the prefilter threshold, Marching Tetrahedra) is computed
//    in FP64 with the reference's operation order and NO fused multiply-add: the
//    reference is gcc -O2 on x86-64 without -march, which never contracts.  The
//    __d*_rn intrinsics are never contracted by nvcc.
//  * Compositing records are FP32; exactness of their inside/outside decisions is kept
//    by an error-bounded filter with an exact FP64 fallback (see composite.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Bounds assertions of the checked build (tools/ab_build.py checked:TS_BOUNDS_CHECKS=1; the
// pool has no compute-sanitizer): a violated index prints its site and traps the context.
#ifdef TS_BOUNDS_CHECKS
#include <cstdio>
#define TS_ASSERT(cond)                                                                     \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("TS_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                           \
      asm volatile("trap;");                                                                \
    }                                                                                       \
  } while (0)
#else
#define TS_ASSERT(cond) \
  do {                  \
  } while (0)
#endif

#define TS_TILE 16
#define TS_TILE_PX (TS_TILE * TS_TILE)

namespace ts {

// ---- exact FP64 arithmetic (no contraction) ----------------------------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ---- camera (camera.py:13-67) -------------------------------------------------------
struct Camera {
  double R[9];  // world -> camera rotation, row major
  double t[3];
  double fx, fy, cx, cy, near_, far_;
  int32_t width, height;
  int32_t pad[2];
};

// ---- fast unsigned division by a runtime constant (a < 2^31) --------------------------
struct FastDiv {
  uint32_t d, mul, shr;
  __host__ __device__ void init(uint32_t den) {
    d = den;
    if (den <= 1) {
      mul = 0;
      shr = 0;
      return;
    }
    uint32_t l = 0;
    while ((1u << l) < den) ++l;  // ceil(log2(den))
    uint32_t p = 31 + l;
    mul = (uint32_t)(((1ull << p) + den - 1) / den);
    shr = p - 32;
  }
  __device__ __forceinline__ uint32_t div(uint32_t a) const { return d <= 1 ? a : (__umulhi(a, mul) >> shr); }
};

// ---- implicit Kuhn grid (grid.py:64-117) --------------------------------------------
// Vertex id = x + n*y + n^2*z (n = R+1); tet id = cell*6 + p, cell = ix*R^2 + iy*R + iz.
// Corners: c0 = 0, c1 = e[P0], c2 = c1 + e[P1], c3 = (1,1,1) with the axis permutations
// of grid.py:18; odd permutations (p = 1, 2, 5) have negative volume and swap v2<->v3
// (grid.py:100-102).  32-bit ids cover R <= 256 (100.7 M tets, 16.97 M vertices).
struct Grid {
  int R, n;
  double step;  // 2.0 / R, numpy linspace's step (delta / div)
  FastDiv dR, dn;
};

inline Grid make_grid(int R) {
  Grid g;
  g.R = R;
  g.n = R + 1;
  g.step = 2.0 / (double)R;
  g.dR.init((uint32_t)R);
  g.dn.init((uint32_t)(R + 1));
  return g;
}

// first / second axis of permutation p: (0,1,2),(0,2,1),(1,0,2),(1,2,0),(2,0,1),(2,1,0)
__host__ __device__ __forceinline__ int perm_a0(int p) { return (p < 2) ? 0 : (p < 4 ? 1 : 2); }
__host__ __device__ __forceinline__ int perm_a1(int p) {
  return (p == 0 || p == 5) ? 1 : ((p == 1 || p == 3) ? 2 : 0);
}
// cell corner (bit 0 = +x, bit 1 = +y, bit 2 = +z) of local slot `slot` of permutation p
// (tet_corners: slot 1 = +a0, slot 2 = +a0+a1, slot 3 = +xyz; odd permutations swap 2 and 3)
__host__ __device__ constexpr int perm_corner(int p, int slot) {
  return slot == 0 ? 0
                   : (slot == 1 ? (1 << perm_a0(p))
                                : (((slot == 2) != (p == 1 || p == 2 || p == 5)) ? ((1 << perm_a0(p)) | (1 << perm_a1(p)))
                                                                                 : 7));
}

// integer vertex coordinates + ids of tet t (local order of grid.py, orientation fixed)
__device__ __forceinline__ void tet_corners(uint32_t t, const Grid& G, int xyz[4][3], uint32_t vid[4]) {
  const uint32_t cell = t / 6u;
  const int p = (int)(t - cell * 6u);
  const uint32_t q = G.dR.div(cell);  // ix*R + iy
  const int iz = (int)(cell - q * (uint32_t)G.R);
  const uint32_t ix = G.dR.div(q);
  const int iy = (int)(q - ix * (uint32_t)G.R);
  const int a0 = perm_a0(p), a1 = perm_a1(p);
  const bool odd = (p == 1 || p == 2 || p == 5);
  // corner offsets without dynamic register indexing (no local memory)
  const int c1x = a0 == 0, c1y = a0 == 1, c1z = a0 == 2;
  const int c2x = c1x | (a1 == 0), c2y = c1y | (a1 == 1), c2z = c1z | (a1 == 2);
  const int b[3] = {(int)ix, iy, iz};
  xyz[0][0] = b[0]; xyz[0][1] = b[1]; xyz[0][2] = b[2];
  xyz[1][0] = b[0] + c1x; xyz[1][1] = b[1] + c1y; xyz[1][2] = b[2] + c1z;
  const int ex = odd ? 1 : c2x, ey = odd ? 1 : c2y, ez = odd ? 1 : c2z;  // slot 2
  const int fx = odd ? c2x : 1, fy = odd ? c2y : 1, fz = odd ? c2z : 1;  // slot 3
  xyz[2][0] = b[0] + ex; xyz[2][1] = b[1] + ey; xyz[2][2] = b[2] + ez;
  xyz[3][0] = b[0] + fx; xyz[3][1] = b[1] + fy; xyz[3][2] = b[2] + fz;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    vid[k] = (uint32_t)xyz[k][0] + (uint32_t)G.n * ((uint32_t)xyz[k][1] + (uint32_t)G.n * (uint32_t)xyz[k][2]);
}

__device__ __forceinline__ void tet_vertices(uint32_t t, const Grid& G, uint32_t vid[4]) {
  int xyz[4][3];
  tet_corners(t, G, xyz, vid);
}

// rest coordinate along one axis: np.linspace(-1, 1, R+1)[i] = i*step + (-1), last = 1
__device__ __forceinline__ double grid_coord(int i, const Grid& G) {
  return i == G.R ? 1.0 : dadd(dmul((double)i, G.step), -1.0);
}

__device__ __forceinline__ void vertex_xyz(uint32_t vid, const Grid& G, int& x, int& y, int& z) {
  const uint32_t q = G.dn.div(vid);  // y + n*z
  x = (int)(vid - q * (uint32_t)G.n);
  const uint32_t zz = G.dn.div(q);
  y = (int)(q - zz * (uint32_t)G.n);
  z = (int)zz;
}

__device__ __forceinline__ void vertex_pos_xyz(const int xyz[3], uint32_t vid, const Grid& G,
                                               const double* __restrict__ deform, double p[3]) {
  p[0] = dadd(grid_coord(xyz[0], G), deform[(size_t)vid * 3 + 0]);
  p[1] = dadd(grid_coord(xyz[1], G), deform[(size_t)vid * 3 + 1]);
  p[2] = dadd(grid_coord(xyz[2], G), deform[(size_t)vid * 3 + 2]);
}

__device__ __forceinline__ void vertex_position(uint32_t vid, const Grid& G, const double* __restrict__ deform,
                                                double p[3]) {
  int xyz[3];
  vertex_xyz(vid, G, xyz[0], xyz[1], xyz[2]);
  vertex_pos_xyz(xyz, vid, G, deform, p);
}

// tet positions + SDF samples (deformed positions, field.py:44-45)
__device__ __forceinline__ void load_tet(uint32_t t, const Grid& G, const double* __restrict__ sdf,
                                         const double* __restrict__ deform, uint32_t v[4], double P[4][3],
                                         double f[4]) {
  int xyz[4][3];
  tet_corners(t, G, xyz, v);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    vertex_pos_xyz(xyz[c], v[c], G, deform, P[c]);
    f[c] = sdf[v[c]];
  }
}

// camera.py:56-67.  p_cam = R p + t (row dot products, left to right), then the pinhole.
__device__ __forceinline__ void project_point(const Camera& c, const double p[3], double& px,
                                              double& py, double& z, double pc[3]) {
  for (int r = 0; r < 3; ++r)
    pc[r] = dadd(dadd(dadd(dmul(p[0], c.R[r * 3 + 0]), dmul(p[1], c.R[r * 3 + 1])),
                      dmul(p[2], c.R[r * 3 + 2])),
                 c.t[r]);
  z = pc[2];
  double zs = z > 1e-12 ? z : 1e-12;
  px = dadd(ddiv(dmul(c.fx, pc[0]), zs), c.cx);
  py = dadd(ddiv(dmul(c.fy, pc[1]), zs), c.cy);
}

// In-tet field gradient, cross-product form (_core.pyx:474-514); returns det = 6V.
__device__ __forceinline__ double tet_gradient(const double P[4][3], const double f[4], double g[3],
                                               double c1[3], double c2[3], double c3[3]) {
  double e1[3], e2[3], e3[3];
  for (int i = 0; i < 3; ++i) {
    e1[i] = dsub(P[1][i], P[0][i]);
    e2[i] = dsub(P[2][i], P[0][i]);
    e3[i] = dsub(P[3][i], P[0][i]);
  }
  c1[0] = dsub(dmul(e2[1], e3[2]), dmul(e2[2], e3[1]));
  c1[1] = dsub(dmul(e2[2], e3[0]), dmul(e2[0], e3[2]));
  c1[2] = dsub(dmul(e2[0], e3[1]), dmul(e2[1], e3[0]));
  c2[0] = dsub(dmul(e3[1], e1[2]), dmul(e3[2], e1[1]));
  c2[1] = dsub(dmul(e3[2], e1[0]), dmul(e3[0], e1[2]));
  c2[2] = dsub(dmul(e3[0], e1[1]), dmul(e3[1], e1[0]));
  c3[0] = dsub(dmul(e1[1], e2[2]), dmul(e1[2], e2[1]));
  c3[1] = dsub(dmul(e1[2], e2[0]), dmul(e1[0], e2[2]));
  c3[2] = dsub(dmul(e1[0], e2[1]), dmul(e1[1], e2[0]));
  double det = dadd(dadd(dmul(e1[0], c1[0]), dmul(e1[1], c1[1])), dmul(e1[2], c1[2]));
  g[0] = g[1] = g[2] = 0.0;
  if (det != 0.0) {
    double d1 = dsub(f[1], f[0]), d2 = dsub(f[2], f[0]), d3 = dsub(f[3], f[0]);
    for (int i = 0; i < 3; ++i)
      g[i] = ddiv(dadd(dadd(dmul(d1, c1[i]), dmul(d2, c2[i])), dmul(d3, c3[i])), det);
  }
  return det;
}

// softplus with the x > 30 passthrough (splat.py:26-28, _core.pyx:29-32)
__device__ __forceinline__ double softplus_d(double x) { return x > 30.0 ? x : log1p(exp(x)); }

// ---- warp / block utilities ----------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// ---- deterministic (fixed-point) gradient accumulation ---------------------------------
// The reference merges per-chunk private buffers in a fixed order (raster.py:217-247), so its
// gradients are bitwise reproducible.  The deterministic mode adds every contribution as a
// 64-bit integer v * 2^36 (integer addition is associative: the sum is independent of the
// order the atomics land in, across CTAs, streams and — all-reduced as int64 — ranks).
// Resolution 2^-36 ~ 1.5e-11 (three orders below Adam's eps = 1e-8), range per contribution
// |v| < 2^26; contributions outside it (or non-finite) are counted in `bad` and dropped.
constexpr double kFxScale = 68719476736.0;           // 2^36
constexpr double kFxInv = 1.4551915228366852e-11;    // 2^-36
constexpr double kFxMax = 67108864.0;                // 2^26

__device__ __forceinline__ void fx_add(long long* addr, double v, unsigned long long* bad) {
  if (v == 0.0) return;
  if (!(fabs(v) < kFxMax)) {  // also NaN
    atomicAdd(bad, 1ull);
    return;
  }
  atomicAdd(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double2ll_rn(v * kFxScale));
}

__device__ __forceinline__ void fx_add4(long long* addr, double a, double b, double c, double d,
                                        unsigned long long* bad) {
  fx_add(addr, a, bad);
  fx_add(addr + 1, b, bad);
  fx_add(addr + 2, c, bad);
  fx_add(addr + 3, d, bad);
}

__device__ __forceinline__ float fx_value(long long v) { return (float)((double)v * kFxInv); }

}  // namespace ts
