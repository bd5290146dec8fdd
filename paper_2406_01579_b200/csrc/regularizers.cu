// regularizers.cu — K8 eikonal + normal-consistency losses and their vertex gradients.
//
// eikonal (_core.pyx:544-568, losses.py:25-36): one thread per tet of the active set,
// FP64 cross-product gradient, (|g|-1)^2, chain to the 4 vertices scattered with one
// red.global.add.v4.f32 per (tet, vertex) into the shared FP32 [N,4] gradient buffer
// (scaled by lambda: the fit loop's weighting, fit.py:196-207, fused here).
//
// normal consistency (_core.pyx:571-668, losses.py:39-52): two per-tet passes and three
// vertex-centric GATHER passes over the implicit Kuhn grid (no atomics, deterministic):
//   T1: per tet, unit normal g/|g| (or "undefined")                        [6R^3 threads]
//   A : vertex mean of incident unit tet normals -> unit vertex normal (+ count, |mean|)
//   B : per-vertex edge term  d_n(v) = -sum_{edge neighbours} n(b), projected back
//       through the normalisation; per-vertex share of sum_edges (1 - n_a.n_b)
//   T2: per tet, the chain through the tet normal: dL/df (4) and g            [6R^3 threads]
//   C : per-vertex sum over incident tets of dL/df_slot and -dL/df_slot * g (the per-tet chain
//       terms are stored in FP32 — they only feed the FP32 gradient buffer; sums in FP64)
// Each tet's FP64 work is done once (not once per incident vertex), and incident tets are
// visited in increasing tet id and edge neighbours in increasing vertex id — the
// reference's accumulation order — so the vertex normals and edge terms are bit-identical to
// the Cython kernel's FP64 values (only the scalar loss is summed in a different order).
#include "internal.cuh"

namespace ts {

constexpr double kEpsNormal = 1e-8;  // field.py:11

// _chain_dg (_core.pyx:517-541): dfs[c] = dL/df_c ; position grad = -dfs[c] * g
__device__ __forceinline__ void chain_coeffs(double det, const double c1[3], const double c2[3], const double c3[3],
                                             const double dg[3], double dfs[4]) {
  double d1 = ddiv(dadd(dadd(dmul(c1[0], dg[0]), dmul(c1[1], dg[1])), dmul(c1[2], dg[2])), det);
  double d2 = ddiv(dadd(dadd(dmul(c2[0], dg[0]), dmul(c2[1], dg[1])), dmul(c2[2], dg[2])), det);
  double d3 = ddiv(dadd(dadd(dmul(c3[0], dg[0]), dmul(c3[1], dg[1])), dmul(c3[2], dg[2])), det);
  dfs[0] = -dadd(dadd(d1, d2), d3);
  dfs[1] = d1;
  dfs[2] = d2;
  dfs[3] = d3;
}

__device__ __forceinline__ double gnorm3(const double g[3]) {
  return sqrt(dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2])));
}

template <typename T>
__device__ __forceinline__ void block_add_to(T v, T* out) {
  v = warp_sum(v);
  __shared__ T ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    atomicAdd(out, t);
  }
}

__global__ void __launch_bounds__(256) k_eikonal(int64_t n, const int32_t* __restrict__ tet_set, Grid G,
                                                 const double* __restrict__ sdf, const double* __restrict__ deform,
                                                 float scale, float* __restrict__ d_vert, double* __restrict__ loss) {
  double local = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v[4];
    double P[4][3], f[4], g[3], c1[3], c2[3], c3[3];
    load_tet((uint32_t)tet_set[i], G, sdf, deform, v, P, f);
    double det = tet_gradient(P, f, g, c1, c2, c3);
    double nrm = gnorm3(g);
    local += dmul(dsub(nrm, 1.0), dsub(nrm, 1.0));
    if (nrm > kEpsNormal && det != 0.0) {
      double w = ddiv(dmul(2.0, dsub(nrm, 1.0)), nrm);
      double dg[3] = {dmul(w, g[0]), dmul(w, g[1]), dmul(w, g[2])};
      double dfs[4];
      chain_coeffs(det, c1, c2, c3, dg, dfs);
      for (int c = 0; c < 4; ++c)
        red_add_v4(d_vert + (size_t)v[c] * 4, (float)(scale * dfs[c]), (float)(-scale * dfs[c] * g[0]),
                   (float)(-scale * dfs[c] * g[1]), (float)(-scale * dfs[c] * g[2]));
    }
  }
  block_add_to(local, loss);
}

// Incident tets of vertex (x,y,z) in increasing tet id.  Calls fn(buffer index, local slot),
// buffer index = x-fastest cell index * 6 + p (see nc_tet_id).
template <class Fn>
__device__ __forceinline__ void for_incident_tets(uint32_t vid, const Grid& G, Fn&& fn) {
  const int R = G.R;
  int x, y, z;
  vertex_xyz(vid, G, x, y, z);
  for (int dx = 1; dx >= 0; --dx)
    for (int dy = 1; dy >= 0; --dy)
      for (int dz = 1; dz >= 0; --dz) {
        const int cx = x - dx, cy = y - dy, cz = z - dz;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= R || cy >= R || cz >= R) continue;
        const int lc = dx | (dy << 1) | (dz << 2);
        // per-tet NC buffers are laid out x-fastest (like vertex ids), not in tet-id order, so
        // neighbouring vertices read neighbouring cells
        const uint32_t cell = ((uint32_t)cz * (uint32_t)R + (uint32_t)cy) * (uint32_t)R + (uint32_t)cx;
        for (int p = 0; p < 6; ++p) {
          const int k1 = 1 << perm_a0(p), k2 = k1 | (1 << perm_a1(p));
          if (lc == 0 || lc == 7 || lc == k1 || lc == k2) {
            // local slot of the vertex in the tet (tet_corners: odd permutations swap 2 and 3)
            const bool odd = (p == 1 || p == 2 || p == 5);
            const int slot = lc == 0 ? 0 : (lc == k1 ? 1 : ((lc == k2) != odd ? 2 : 3));
            fn(cell * 6u + (uint32_t)p, slot);
          }
        }
      }
}

// tet id of per-tet NC buffer index i (cells x-fastest there, z-fastest in tet ids)
__device__ __forceinline__ uint32_t nc_tet_id(int64_t i, const Grid& G) {
  const uint32_t cell = (uint32_t)(i / 6), p = (uint32_t)(i - (int64_t)cell * 6);
  const uint32_t q = G.dR.div(cell);  // cy + R cz
  const uint32_t cx = cell - q * (uint32_t)G.R;
  const uint32_t cz = G.dR.div(q);
  const uint32_t cy = q - cz * (uint32_t)G.R;
  return ((cx * (uint32_t)G.R + cy) * (uint32_t)G.R + cz) * 6u + p;
}

// pass T1: per-tet unit normal (w = 1) or undefined (all 0)
__global__ void __launch_bounds__(256) k_nc_tet_normals(int64_t T, Grid G, const double* __restrict__ sdf,
                                                        const double* __restrict__ deform, double4* __restrict__ tn) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v[4];
    double P[4][3], f[4], g[3], c1[3], c2[3], c3[3];
    load_tet(nc_tet_id(t, G), G, sdf, deform, v, P, f);
    tet_gradient(P, f, g, c1, c2, c3);
    const double nrm = gnorm3(g);
    tn[t] = nrm < kEpsNormal ? make_double4(0.0, 0.0, 0.0, 0.0)
                             : make_double4(ddiv(g[0], nrm), ddiv(g[1], nrm), ddiv(g[2], nrm), 1.0);
  }
}

// pass A: nv = normalized mean of incident unit normals; cnt; an (0 = undefined)
__global__ void __launch_bounds__(256) k_nc_vertex_normals(int64_t N, Grid G, const double4* __restrict__ tn,
                                                           double* __restrict__ nv, double* __restrict__ cnt,
                                                           double* __restrict__ an) {
  for (int64_t vid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vid < N;
       vid += (int64_t)gridDim.x * blockDim.x) {
    double s[3] = {0.0, 0.0, 0.0}, c = 0.0;
    for_incident_tets((uint32_t)vid, G, [&](uint32_t t, int) {
      const double4 q = tn[t];
      if (q.w == 0.0) return;
      c = dadd(c, 1.0);
      s[0] = dadd(s[0], q.x);
      s[1] = dadd(s[1], q.y);
      s[2] = dadd(s[2], q.z);
    });
    double a = 0.0;
    if (c != 0.0) {
      for (int i = 0; i < 3; ++i) s[i] = ddiv(s[i], c);
      double m = gnorm3(s);
      if (!(m < kEpsNormal)) {
        a = m;
        for (int i = 0; i < 3; ++i) s[i] = ddiv(s[i], m);
      }
    }
    for (int i = 0; i < 3; ++i) nv[vid * 3 + i] = s[i];
    cnt[vid] = c != 0.0 ? ddiv(1.0, c) : 0.0;  // stored as the reciprocal the chain pass uses
    an[vid] = a;
  }
}

// pass B: edge penalty and its gradient, pushed back through the vertex normalisation
__global__ void __launch_bounds__(256) k_nc_edges(int64_t N, Grid G, const double* __restrict__ nv,
                                                  const double* __restrict__ an, double* __restrict__ dm,
                                                  double* __restrict__ loss) {
  const int64_t n = G.n;
  // Kuhn edge offsets (grid.py:106-107) as vertex-id deltas, ascending
  const int64_t off[7] = {1, n, n + 1, n * n, n * n + 1, n * n + n, n * n + n + 1};
  const int ox[7] = {1, 0, 1, 0, 1, 0, 1}, oy[7] = {0, 1, 1, 0, 0, 1, 1}, oz[7] = {0, 0, 0, 1, 1, 1, 1};
  double local = 0.0;
  for (int64_t vid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vid < N;
       vid += (int64_t)gridDim.x * blockDim.x) {
    int x, y, z;
    vertex_xyz((uint32_t)vid, G, x, y, z);
    double d[3] = {0.0, 0.0, 0.0};
    const bool def = an[vid] != 0.0;
    const double a0 = nv[vid * 3], a1 = nv[vid * 3 + 1], a2 = nv[vid * 3 + 2];
    // lower neighbours (ascending id = descending delta), then upper ones
    for (int e = 6; e >= 0; --e) {
      if (x - ox[e] < 0 || y - oy[e] < 0 || z - oz[e] < 0) continue;
      const int64_t b = vid - off[e];
      if (!def || an[b] == 0.0) continue;
      for (int i = 0; i < 3; ++i) d[i] = dsub(d[i], nv[b * 3 + i]);
    }
    for (int e = 0; e < 7; ++e) {
      if (x + ox[e] >= n || y + oy[e] >= n || z + oz[e] >= n) continue;
      const int64_t b = vid + off[e];
      if (!def || an[b] == 0.0) continue;
      const double b0 = nv[b * 3], b1 = nv[b * 3 + 1], b2 = nv[b * 3 + 2];
      local += dsub(1.0, dadd(dadd(dmul(a0, b0), dmul(a1, b1)), dmul(a2, b2)));
      d[0] = dsub(d[0], b0);
      d[1] = dsub(d[1], b1);
      d[2] = dsub(d[2], b2);
    }
    if (def) {
      double dot = dadd(dadd(dmul(a0, d[0]), dmul(a1, d[1])), dmul(a2, d[2]));
      const double av = an[vid];
      d[0] = ddiv(dsub(d[0], dmul(a0, dot)), av);
      d[1] = ddiv(dsub(d[1], dmul(a1, dot)), av);
      d[2] = ddiv(dsub(d[2], dmul(a2, dot)), av);
    }
    for (int i = 0; i < 3; ++i) dm[vid * 3 + i] = d[i];
  }
  block_add_to(local, loss);
}

// pass T2: per-tet chain through the tet normal (_core.pyx:651-667): dL/df per slot and g
// (zeros where the reference skips the tet)
__global__ void __launch_bounds__(256) k_nc_tet_chain(int64_t T, Grid G, const double* __restrict__ sdf,
                                                      const double* __restrict__ deform,
                                                      const double* __restrict__ icnt, const double* __restrict__ dm,
                                                      float4* __restrict__ tdf, float4* __restrict__ tg) {
  // FP64 throughout, but with reciprocals instead of the reference's repeated divisions: the
  // results are rounded to FP32 for the gradient buffer anyway (the skip tests are unchanged)
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v[4];
    double P[4][3], f[4];
    load_tet(nc_tet_id(t, G), G, sdf, deform, v, P, f);
    double e1[3], e2[3], e3[3], c1[3], c2[3], c3[3];
    for (int i = 0; i < 3; ++i) {
      e1[i] = P[1][i] - P[0][i];
      e2[i] = P[2][i] - P[0][i];
      e3[i] = P[3][i] - P[0][i];
    }
    c1[0] = e2[1] * e3[2] - e2[2] * e3[1];
    c1[1] = e2[2] * e3[0] - e2[0] * e3[2];
    c1[2] = e2[0] * e3[1] - e2[1] * e3[0];
    c2[0] = e3[1] * e1[2] - e3[2] * e1[1];
    c2[1] = e3[2] * e1[0] - e3[0] * e1[2];
    c2[2] = e3[0] * e1[1] - e3[1] * e1[0];
    c3[0] = e1[1] * e2[2] - e1[2] * e2[1];
    c3[1] = e1[2] * e2[0] - e1[0] * e2[2];
    c3[2] = e1[0] * e2[1] - e1[1] * e2[0];
    const double det = e1[0] * c1[0] + e1[1] * c1[1] + e1[2] * c1[2];
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f), og = make_float4(0.f, 0.f, 0.f, 0.f);
    if (det != 0.0) {
      const double idet = 1.0 / det;
      const double d1 = f[1] - f[0], d2 = f[2] - f[0], d3 = f[3] - f[0];
      double g[3];
      for (int i = 0; i < 3; ++i) g[i] = (d1 * c1[i] + d2 * c2[i] + d3 * c3[i]) * idet;
      const double nrm = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
      if (!(nrm < kEpsNormal)) {
        const double inrm = 1.0 / nrm;
        const double nt[3] = {g[0] * inrm, g[1] * inrm, g[2] * inrm};
        double dnt[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < 4; ++c) {
          const double inv = icnt[v[c]];
          for (int i = 0; i < 3; ++i) dnt[i] += dm[v[c] * 3 + i] * inv;
        }
        const double dot = nt[0] * dnt[0] + nt[1] * dnt[1] + nt[2] * dnt[2];
        double dg[3];
        for (int i = 0; i < 3; ++i) dg[i] = (dnt[i] - nt[i] * dot) * inrm;
        const double k1 = (c1[0] * dg[0] + c1[1] * dg[1] + c1[2] * dg[2]) * idet;
        const double k2 = (c2[0] * dg[0] + c2[1] * dg[1] + c2[2] * dg[2]) * idet;
        const double k3 = (c3[0] * dg[0] + c3[1] * dg[1] + c3[2] * dg[2]) * idet;
        o = make_float4((float)(-(k1 + k2 + k3)), (float)k1, (float)k2, (float)k3);
        og = make_float4((float)g[0], (float)g[1], (float)g[2], 1.f);
      }
    }
    tdf[t] = o;
    tg[t] = og;
  }
}

// pass C: per-vertex gather of the per-tet chain terms
__global__ void __launch_bounds__(256) k_nc_grad(int64_t N, Grid G, const float4* __restrict__ tdf,
                                                 const float4* __restrict__ tg, float scale,
                                                 float* __restrict__ d_vert) {
  for (int64_t vid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vid < N;
       vid += (int64_t)gridDim.x * blockDim.x) {
    double ds = 0.0, dp[3] = {0.0, 0.0, 0.0};
    for_incident_tets((uint32_t)vid, G, [&](uint32_t t, int slot) {
      const float4 gq = tg[t];
      if (gq.w == 0.f) return;  // skipped by the reference (undefined normal or det == 0)
      const float4 dq = tdf[t];
      const double d = slot == 0 ? dq.x : (slot == 1 ? dq.y : (slot == 2 ? dq.z : dq.w));
      ds = dadd(ds, d);
      dp[0] = dsub(dp[0], dmul(d, gq.x));
      dp[1] = dsub(dp[1], dmul(d, gq.y));
      dp[2] = dsub(dp[2], dmul(d, gq.z));
    });
    // atomic add: the fit step runs the regularizers concurrently with the views' chains
    red_add_v4(d_vert + vid * 4, (float)(scale * ds), (float)(scale * dp[0]), (float)(scale * dp[1]),
               (float)(scale * dp[2]));
  }
}

// Adam (fit.py:70-90) on the interleaved FP32 gradient buffer: FP64 moments and parameters,
// torch's operation order (m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// p -= lr (m/c1) / (sqrt(v/c2) + eps)), deformation clamped to +-limit afterwards.
__global__ void __launch_bounds__(256) k_adam(int64_t N, const float4* __restrict__ g4, double* __restrict__ sdf,
                                              double* __restrict__ deform, double* __restrict__ m_sdf,
                                              double* __restrict__ v_sdf, double* __restrict__ m_def,
                                              double* __restrict__ v_def, double lr_sdf, double lr_def, double b1,
                                              double b2, double c1, double c2, double eps, double limit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 g = g4[i];
    const double gs[4] = {(double)g.x, (double)g.y, (double)g.z, (double)g.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double* p = c == 0 ? sdf + i : deform + 3 * i + (c - 1);
      double* m = c == 0 ? m_sdf + i : m_def + 3 * i + (c - 1);
      double* v = c == 0 ? v_sdf + i : v_def + 3 * i + (c - 1);
      const double lr = c == 0 ? lr_sdf : lr_def;
      const double mm = dadd(dmul(*m, b1), dmul(gs[c], 1.0 - b1));
      const double vv = dadd(dmul(*v, b2), dmul(dmul(gs[c], gs[c]), 1.0 - b2));
      *m = mm;
      *v = vv;
      double np = dsub(*p, dmul(lr, ddiv(ddiv(mm, c1), dadd(sqrt(ddiv(vv, c2)), eps))));
      if (c > 0) np = fmin(fmax(np, -limit), limit);
      *p = np;
    }
  }
}

}  // namespace ts

using namespace ts;

void ts_impl_adam(int64_t N, const float* g4, double* sdf, double* deform, double* m_sdf, double* v_sdf,
                  double* m_def, double* v_def, double lr_sdf, double lr_def, double b1, double b2, int64_t t,
                  double eps, double limit, cudaStream_t st) {
  if (N <= 0) return;
  const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
  int blocks = (int)((N + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_adam<<<blocks, 256, 0, st>>>(N, reinterpret_cast<const float4*>(g4), sdf, deform, m_sdf, v_sdf, m_def, v_def,
                                 lr_sdf, lr_def, b1, b2, c1, c2, eps, limit);
}

void ts_impl_eikonal(const double* sdf, const double* deform, int R, const int32_t* tet_set, int64_t n, float scale,
                     float* d_vert, double* loss, cudaStream_t st) {
  cudaMemsetAsync(loss, 0, sizeof(double), st);
  if (n <= 0) return;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_eikonal<<<blocks, 256, 0, st>>>(n, tet_set, make_grid(R), sdf, deform, scale, d_vert, loss);
}

// scratch layout of the normal-consistency passes (16-byte aligned pieces)
static void nc_layout(int R, int64_t off[8]) {
  const int64_t n = R + 1, N = n * n * n, T = 6 * (int64_t)R * R * R;
  const int64_t sz[7] = {24 * N, 24 * N, 8 * N, 8 * N, 32 * T, 16 * T, 16 * T};  // nv dm cnt an tn tdf tg
  off[0] = 0;
  for (int i = 0; i < 7; ++i) off[i + 1] = off[i] + ((sz[i] + 255) & ~255ll);
}

int64_t ts_impl_nc_scratch_bytes(int R) {
  int64_t off[8];
  nc_layout(R, off);
  return off[7];
}

// scratch: ts_impl_nc_scratch_bytes(R) bytes of device memory, or nullptr (stream-ordered pool)
void ts_impl_normal_consistency(const double* sdf, const double* deform, int R, float scale, float* d_vert,
                                double* loss, cudaStream_t st, void* scratch) {
  const int64_t n = R + 1, N = n * n * n, T = 6 * (int64_t)R * R * R;
  cudaMemsetAsync(loss, 0, sizeof(double), st);
  int64_t off[8];
  nc_layout(R, off);
  char* base = static_cast<char*>(scratch);
  if (!base) cudaMallocAsync(reinterpret_cast<void**>(&base), off[7], st);
  double* nv = reinterpret_cast<double*>(base + off[0]);
  double* dm = reinterpret_cast<double*>(base + off[1]);
  double* cnt = reinterpret_cast<double*>(base + off[2]);
  double* an = reinterpret_cast<double*>(base + off[3]);
  double4* tn = reinterpret_cast<double4*>(base + off[4]);  // T1: unit tet normals (FP64: they feed the loss)
  float4* tdf = reinterpret_cast<float4*>(base + off[5]);   // T2: per-tet chain terms (FP32: gradient only)
  float4* tg = reinterpret_cast<float4*>(base + off[6]);
  const Grid G = make_grid(R);
  const int vblocks = (int)((N + 255) / 256 < 148 * 8 ? (N + 255) / 256 : 148 * 8);
  const int tblocks = (int)((T + 255) / 256 < 148 * 16 ? (T + 255) / 256 : 148 * 16);
  k_nc_tet_normals<<<tblocks, 256, 0, st>>>(T, G, sdf, deform, tn);
  k_nc_vertex_normals<<<vblocks, 256, 0, st>>>(N, G, tn, nv, cnt, an);
  k_nc_edges<<<vblocks, 256, 0, st>>>(N, G, nv, an, dm, loss);
  k_nc_tet_chain<<<tblocks, 256, 0, st>>>(T, G, sdf, deform, cnt, dm, tdf, tg);
  k_nc_grad<<<vblocks, 256, 0, st>>>(N, G, tdf, tg, scale, d_vert);
  if (!scratch) cudaFreeAsync(base, st);
}
