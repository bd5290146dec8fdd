// meshraster.cu — z-buffered flat-shaded rasterization of a triangle mesh (mesh.py:98-147),
// the surface-limit reference the splatted maps are compared with.
//
// The reference walks the triangles in order and keeps, per pixel, the first triangle with
// the strictly smallest perspective-correct depth.  Here every triangle is a thread over its
// pixel box; three passes make the result order-independent and identical:
//   1. per-pixel atomicMin of the FP64 depth (positive doubles order as their bit patterns),
//   2. among the triangles reaching that depth, atomicMin of the triangle index,
//   3. per pixel: mask, depth, and the winner's unit face normal.
// All per-pixel arithmetic is the reference's FP64 operation sequence (no contraction).
#include "internal.cuh"

namespace ts {

constexpr int64_t kMeshNone = 0x7f7f7f7f7f7f7f7fll;  // memset(0x7f) sentinel: no triangle

struct MeshTri {
  double ax, ay, bx, by, cx, cy, za, zb, zc, det;
  int x0, x1, y0, y1;
};

// projection + the reference's per-triangle rejections and pixel box; false = skip
__device__ __forceinline__ bool mesh_tri(int64_t t, const int64_t* __restrict__ tris, const double* __restrict__ pix,
                                         const double* __restrict__ z, const double* __restrict__ verts,
                                         const Camera& cam, MeshTri& m) {
  const int64_t i0 = tris[3 * t], i1 = tris[3 * t + 1], i2 = tris[3 * t + 2];
  m.za = z[i0];
  m.zb = z[i1];
  m.zc = z[i2];
  const double zmin = fmin(fmin(m.za, m.zb), m.zc), zmax = fmax(fmax(m.za, m.zb), m.zc);
  const double* A = verts + 3 * i0;
  const double* B = verts + 3 * i1;
  const double* C = verts + 3 * i2;
  const double e1[3] = {dsub(B[0], A[0]), dsub(B[1], A[1]), dsub(B[2], A[2])};
  const double e2[3] = {dsub(C[0], A[0]), dsub(C[1], A[1]), dsub(C[2], A[2])};
  const double f0 = dsub(dmul(e1[1], e2[2]), dmul(e1[2], e2[1]));
  const double f1 = dsub(dmul(e1[2], e2[0]), dmul(e1[0], e2[2]));
  const double f2 = dsub(dmul(e1[0], e2[1]), dmul(e1[1], e2[0]));
  const double nrm = sqrt(dadd(dadd(dmul(f0, f0), dmul(f1, f1)), dmul(f2, f2)));
  if (zmin <= cam.near_ || zmax >= cam.far_ || nrm == 0.0) return false;
  m.ax = pix[2 * i0];
  m.ay = pix[2 * i0 + 1];
  m.bx = pix[2 * i1];
  m.by = pix[2 * i1 + 1];
  m.cx = pix[2 * i2];
  m.cy = pix[2 * i2 + 1];
  m.x0 = max((int)floor(fmin(fmin(m.ax, m.bx), m.cx)), 0);
  m.x1 = min((int)ceil(fmax(fmax(m.ax, m.bx), m.cx)), cam.width - 1);
  m.y0 = max((int)floor(fmin(fmin(m.ay, m.by), m.cy)), 0);
  m.y1 = min((int)ceil(fmax(fmax(m.ay, m.by), m.cy)), cam.height - 1);
  if (m.x0 > m.x1 || m.y0 > m.y1) return false;
  m.det = dsub(dmul(dsub(m.bx, m.ax), dsub(m.cy, m.ay)), dmul(dsub(m.cx, m.ax), dsub(m.by, m.ay)));
  return !(fabs(m.det) < 1e-12);
}

// depth of pixel centre (xs, ys) in the triangle, or -1 when outside
__device__ __forceinline__ double mesh_depth(const MeshTri& m, double xs, double ys) {
  const double u = ddiv(dsub(dmul(dsub(xs, m.ax), dsub(m.cy, m.ay)), dmul(dsub(ys, m.ay), dsub(m.cx, m.ax))), m.det);
  const double v = ddiv(dadd(dmul(dsub(xs, m.ax), -dsub(m.by, m.ay)), dmul(dsub(ys, m.ay), dsub(m.bx, m.ax))), m.det);
  if (!(u >= 0.0 && v >= 0.0 && dadd(u, v) <= 1.0)) return -1.0;
  const double denom = dadd(dadd(ddiv(dsub(dsub(1.0, u), v), m.za), ddiv(u, m.zb)), ddiv(v, m.zc));
  return ddiv(1.0, denom);
}

__global__ void k_mesh_project(int64_t V, const double* __restrict__ verts, Camera cam, double* __restrict__ pix,
                               double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    const double p[3] = {verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]};
    double px, py, zz, pc[3];
    project_point(cam, p, px, py, zz, pc);
    pix[2 * i] = px;
    pix[2 * i + 1] = py;
    z[i] = zz;
  }
}

// pass 1 (win == nullptr): depth minimum; pass 2: the smallest triangle index at that depth
__global__ void k_mesh_zpass(int64_t F, const int64_t* __restrict__ tris, const double* __restrict__ verts,
                             const double* __restrict__ pix, const double* __restrict__ z, Camera cam,
                             unsigned long long* __restrict__ zbuf, int64_t* __restrict__ win) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < F; t += (int64_t)gridDim.x * blockDim.x) {
    MeshTri m;
    if (!mesh_tri(t, tris, pix, z, verts, cam, m)) continue;
    for (int y = m.y0; y <= m.y1; ++y)
      for (int x = m.x0; x <= m.x1; ++x) {
        const double zp = mesh_depth(m, x + 0.5, y + 0.5);
        if (zp < 0.0) continue;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(zp);
        const int64_t p = (int64_t)y * cam.width + x;
        if (!win)
          atomicMin(zbuf + p, bits);
        else if (bits == zbuf[p])
          atomicMin(reinterpret_cast<unsigned long long*>(win) + p, (unsigned long long)t);
      }
  }
}

__global__ void k_mesh_resolve(int64_t HW, const int64_t* __restrict__ win, const unsigned long long* __restrict__ zbuf,
                               const int64_t* __restrict__ tris, const double* __restrict__ verts,
                               uint8_t* __restrict__ mask, double* __restrict__ depth, double* __restrict__ normal) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < HW; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = win[p];
    if (t == kMeshNone) {
      mask[p] = 0;
      depth[p] = 0.0;
      normal[3 * p] = normal[3 * p + 1] = normal[3 * p + 2] = 0.0;
      continue;
    }
    const double* A = verts + 3 * tris[3 * t];
    const double* B = verts + 3 * tris[3 * t + 1];
    const double* C = verts + 3 * tris[3 * t + 2];
    const double e1[3] = {dsub(B[0], A[0]), dsub(B[1], A[1]), dsub(B[2], A[2])};
    const double e2[3] = {dsub(C[0], A[0]), dsub(C[1], A[1]), dsub(C[2], A[2])};
    const double f[3] = {dsub(dmul(e1[1], e2[2]), dmul(e1[2], e2[1])), dsub(dmul(e1[2], e2[0]), dmul(e1[0], e2[2])),
                         dsub(dmul(e1[0], e2[1]), dmul(e1[1], e2[0]))};
    const double nrm = sqrt(dadd(dadd(dmul(f[0], f[0]), dmul(f[1], f[1])), dmul(f[2], f[2])));
    mask[p] = 1;
    depth[p] = __longlong_as_double((long long)zbuf[p]);
    for (int c = 0; c < 3; ++c) normal[3 * p + c] = ddiv(f[c], nrm);
  }
}

}  // namespace ts

using namespace ts;

int ts_impl_rasterize_mesh(const double* verts, int64_t V, const int64_t* tris, int64_t F, const Camera& cam,
                           uint8_t* mask, double* depth, double* normal, cudaStream_t st) {
  const int64_t HW = (int64_t)cam.width * cam.height;
  double *pix = nullptr, *z = nullptr;
  unsigned long long* zbuf = nullptr;
  int64_t* win = nullptr;
  cudaMallocAsync(&pix, sizeof(double) * 2 * (V > 0 ? V : 1), st);
  cudaMallocAsync(&z, sizeof(double) * (V > 0 ? V : 1), st);
  cudaMallocAsync(&zbuf, sizeof(unsigned long long) * HW, st);
  cudaMallocAsync(&win, sizeof(int64_t) * HW, st);
  // sentinels 0x7f7f...7f: above the bit pattern of any finite depth and of any triangle index
  cudaMemsetAsync(zbuf, 0x7f, sizeof(unsigned long long) * HW, st);
  cudaMemsetAsync(win, 0x7f, sizeof(int64_t) * HW, st);
  const int vb = (int)((V + 255) / 256 < 4096 ? (V + 255) / 256 : 4096);
  const int fb = (int)((F + 127) / 128 < 4096 ? (F + 127) / 128 : 4096);
  const int pb = (int)((HW + 255) / 256 < 4096 ? (HW + 255) / 256 : 4096);
  if (V > 0) k_mesh_project<<<vb > 0 ? vb : 1, 256, 0, st>>>(V, verts, cam, pix, z);
  if (F > 0) {
    k_mesh_zpass<<<fb, 128, 0, st>>>(F, tris, verts, pix, z, cam, zbuf, nullptr);
  }
  if (F > 0) k_mesh_zpass<<<fb, 128, 0, st>>>(F, tris, verts, pix, z, cam, zbuf, win);
  k_mesh_resolve<<<pb, 256, 0, st>>>(HW, win, zbuf, tris, verts, mask, depth, normal);
  cudaFreeAsync(pix, st);
  cudaFreeAsync(z, st);
  cudaFreeAsync(zbuf, st);
  cudaFreeAsync(win, st);
  return 0;
}
