// regularizers.cu — K8 eikonal + normal-consistency losses and their vertex gradients.
//
// eikonal (_core.pyx:544-568, losses.py:25-36): one thread per tet of the active set,
// FP64 cross-product gradient, (|g|-1)^2, chain to the 4 vertices scattered with one
// red.global.add.v4.f32 per (tet, vertex) into the shared FP32 [N,4] gradient buffer
// (scaled by lambda: the fit loop's weighting, fit.py:196-207, fused here).
//
// normal consistency (_core.pyx:571-668, losses.py:39-52): two per-tet passes and three
// vertex-centric GATHER passes over the implicit Kuhn grid (no atomics, deterministic):
//   T1: per tet, unit normal g/|g| (or "undefined")   [one thread per cell: its 8 corners
//       are loaded once for the cell's 6 tets]
//   A : vertex mean of incident unit tet normals -> unit vertex normal (+ count, |mean|)
//   B : per-vertex edge term  d_n(v) = -sum_{edge neighbours} n(b), projected back
//       through the normalisation; per-vertex share of sum_edges (1 - n_a.n_b)
//   T2: per tet, the chain through the tet normal: dL/df (4) and g   [one thread per cell]
// Per-tet buffers are p-major (index p R^3 + x-fastest cell): T1/T2 store coalesced per
// permutation and the vertex gathers read one contiguous run per (cell offset, p).
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
                                                 float scale, float* __restrict__ d_vert, double* __restrict__ loss,
                                                 Fx fx) {
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
      for (int c = 0; c < 4; ++c) {
        if (fx.vert)
          fx_add4(fx.vert + (size_t)v[c] * 4, scale * dfs[c], -scale * dfs[c] * g[0], -scale * dfs[c] * g[1],
                  -scale * dfs[c] * g[2], fx.bad);
        else
          red_add_v4(d_vert + (size_t)v[c] * 4, (float)(scale * dfs[c]), (float)(-scale * dfs[c] * g[0]),
                     (float)(-scale * dfs[c] * g[1]), (float)(-scale * dfs[c] * g[2]));
      }
    }
  }
  block_add_to(local, loss);
}

// Incident tets of vertex (x,y,z) in increasing tet id.  Calls fn(buffer index, local slot),
// buffer index = p * R^3 + x-fastest cell index (see nc_tet_id).
template <class Fn>
__device__ __forceinline__ void for_incident_tets(uint32_t vid, const Grid& G, Fn&& fn) {
  const int R = G.R;
  int x, y, z;
  vertex_xyz(vid, G, x, y, z);
#pragma unroll
  for (int dx = 1; dx >= 0; --dx)
#pragma unroll
    for (int dy = 1; dy >= 0; --dy)
#pragma unroll
      for (int dz = 1; dz >= 0; --dz) {
        const int cx = x - dx, cy = y - dy, cz = z - dz;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= R || cy >= R || cz >= R) continue;
        const int lc = dx | (dy << 1) | (dz << 2);
        // per-tet NC buffers are p-major with cells x-fastest (like vertex ids), not in tet-id
        // order: a warp of neighbouring vertices reads one contiguous run per (cell offset, p)
        const uint32_t cell = ((uint32_t)cz * (uint32_t)R + (uint32_t)cy) * (uint32_t)R + (uint32_t)cx;
        const uint32_t C = (uint32_t)R * (uint32_t)R * (uint32_t)R;
#pragma unroll
        for (int p = 0; p < 6; ++p) {
          const int k1 = 1 << perm_a0(p), k2 = k1 | (1 << perm_a1(p));
          if (lc == 0 || lc == 7 || lc == k1 || lc == k2) {
            // local slot of the vertex in the tet (tet_corners: odd permutations swap 2 and 3)
            const bool odd = (p == 1 || p == 2 || p == 5);
            const int slot = lc == 0 ? 0 : (lc == k1 ? 1 : ((lc == k2) != odd ? 2 : 3));
            fn((uint32_t)p * C + cell, slot);
          }
        }
      }
}

// The 8 corners of cell (cx, cy, cz) — deformed positions and SDF (corner bit 0 = +x,
// bit 1 = +y, bit 2 = +z), loaded once for the cell's 6 tets.
struct CellCorners {
  double P[8][3], f[8];
  uint32_t v[8];
};
__device__ __forceinline__ void load_cell(uint32_t c, const Grid& G, const double* __restrict__ sdf,
                                          const double* __restrict__ deform, CellCorners& K) {
  const uint32_t q = G.dR.div(c);  // cy + R cz
  const int cx = (int)(c - q * (uint32_t)G.R);
  const uint32_t czu = G.dR.div(q);
  const int cy = (int)(q - czu * (uint32_t)G.R), cz = (int)czu;
#pragma unroll
  for (int lc = 0; lc < 8; ++lc) {
    const int xyz[3] = {cx + (lc & 1), cy + ((lc >> 1) & 1), cz + ((lc >> 2) & 1)};
    K.v[lc] = (uint32_t)xyz[0] + (uint32_t)G.n * ((uint32_t)xyz[1] + (uint32_t)G.n * (uint32_t)xyz[2]);
    vertex_pos_xyz(xyz, K.v[lc], G, deform, K.P[lc]);
    K.f[lc] = __ldg(sdf + K.v[lc]);
  }
}

template <int p>
__device__ __forceinline__ void cell_tet(const CellCorners& K, uint32_t v[4], double P[4][3], double f[4]) {
#pragma unroll
  for (int sl = 0; sl < 4; ++sl) {
    const int lc = perm_corner(p, sl);
    v[sl] = K.v[lc];
    f[sl] = K.f[lc];
#pragma unroll
    for (int i = 0; i < 3; ++i) P[sl][i] = K.P[lc][i];
  }
}

// pass T1: per-tet unit normal (w = 1) or undefined (all 0); one thread per cell, 6 tets
template <int p>
__device__ __forceinline__ void t1_tet(const CellCorners& K, double4* __restrict__ out) {
  uint32_t v[4];
  double P[4][3], f[4], g[3], c1[3], c2[3], c3[3];
  cell_tet<p>(K, v, P, f);
  tet_gradient(P, f, g, c1, c2, c3);
  const double nrm = gnorm3(g);
  *out = nrm < kEpsNormal ? make_double4(0.0, 0.0, 0.0, 0.0)
                          : make_double4(ddiv(g[0], nrm), ddiv(g[1], nrm), ddiv(g[2], nrm), 1.0);
}

// Every pass runs over an index range (cells [c_lo, c_hi) / vertices [lo, hi), contiguous z-slabs
// of the x-fastest ids): a rank computes the gradient of its vertex slab from its slab plus the
// halo layers each pass reads (ts_impl_normal_consistency).
__global__ void __launch_bounds__(256) k_nc_tet_normals(int64_t C, int64_t c_lo, int64_t c_hi, Grid G,
                                                        const double* __restrict__ sdf,
                                                        const double* __restrict__ deform, double4* __restrict__ tn) {
  for (int64_t c = c_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < c_hi;
       c += (int64_t)gridDim.x * blockDim.x) {
    CellCorners K;
    load_cell((uint32_t)c, G, sdf, deform, K);
    t1_tet<0>(K, tn + c);
    t1_tet<1>(K, tn + C + c);
    t1_tet<2>(K, tn + 2 * C + c);
    t1_tet<3>(K, tn + 3 * C + c);
    t1_tet<4>(K, tn + 4 * C + c);
    t1_tet<5>(K, tn + 5 * C + c);
  }
}

// pass A: nv = normalized mean of incident unit normals, .w = |mean| (0 = undefined);
// icnt = 1 / count (0 without a defined incident tet)
__global__ void __launch_bounds__(256) k_nc_vertex_normals(int64_t lo, int64_t hi, Grid G,
                                                           const double4* __restrict__ tn,
                                                           double4* __restrict__ nv, double* __restrict__ icnt) {
  for (int64_t vid = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vid < hi;
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
    nv[vid] = make_double4(s[0], s[1], s[2], a);
    icnt[vid] = c != 0.0 ? ddiv(1.0, c) : 0.0;  // the reciprocal the chain pass uses
  }
}

// pass B: edge penalty and its gradient, pushed back through the vertex normalisation; the
// result is stored pre-multiplied by 1/count (the factor the tet chain applies per vertex).
// Each edge's penalty is counted by its lower vertex, and only for vertices in [llo, lhi)
// (the slab's own vertices: the halo's edges belong to the neighbouring slab).
__global__ void __launch_bounds__(256) k_nc_edges(int64_t lo, int64_t hi, int64_t llo, int64_t lhi, Grid G,
                                                  const double4* __restrict__ nv,
                                                  const double* __restrict__ icnt, double4* __restrict__ dmi,
                                                  double* __restrict__ loss) {
  const int64_t n = G.n;
  // Kuhn edge offsets (grid.py:106-107) as vertex-id deltas, ascending
  const int64_t off[7] = {1, n, n + 1, n * n, n * n + 1, n * n + n, n * n + n + 1};
  const int ox[7] = {1, 0, 1, 0, 1, 0, 1}, oy[7] = {0, 1, 1, 0, 0, 1, 1}, oz[7] = {0, 0, 0, 1, 1, 1, 1};
  double local = 0.0;
  for (int64_t vid = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vid < hi;
       vid += (int64_t)gridDim.x * blockDim.x) {
    int x, y, z;
    vertex_xyz((uint32_t)vid, G, x, y, z);
    const bool own = vid >= llo && vid < lhi;
    double d[3] = {0.0, 0.0, 0.0};
    const double4 A = nv[vid];
    const bool def = A.w != 0.0;
    // neighbour records loaded up front, 7 at a time (independent loads), then the FP64
    // sums in order: lower neighbours (ascending id = descending delta), then upper ones
    double4 nb[7];
#pragma unroll
    for (int e = 0; e < 7; ++e)
      nb[e] = def && x - ox[e] >= 0 && y - oy[e] >= 0 && z - oz[e] >= 0 ? nv[vid - off[e]]
                                                                        : make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
    for (int e = 6; e >= 0; --e) {
      if (nb[e].w == 0.0) continue;
      d[0] = dsub(d[0], nb[e].x);
      d[1] = dsub(d[1], nb[e].y);
      d[2] = dsub(d[2], nb[e].z);
    }
#pragma unroll
    for (int e = 0; e < 7; ++e)
      nb[e] = def && x + ox[e] < n && y + oy[e] < n && z + oz[e] < n ? nv[vid + off[e]]
                                                                     : make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
    for (int e = 0; e < 7; ++e) {
      const double4 B = nb[e];
      if (B.w == 0.0) continue;
      if (own) local += dsub(1.0, dadd(dadd(dmul(A.x, B.x), dmul(A.y, B.y)), dmul(A.z, B.z)));
      d[0] = dsub(d[0], B.x);
      d[1] = dsub(d[1], B.y);
      d[2] = dsub(d[2], B.z);
    }
    if (def) {
      double dot = dadd(dadd(dmul(A.x, d[0]), dmul(A.y, d[1])), dmul(A.z, d[2]));
      d[0] = ddiv(dsub(d[0], dmul(A.x, dot)), A.w);
      d[1] = ddiv(dsub(d[1], dmul(A.y, dot)), A.w);
      d[2] = ddiv(dsub(d[2], dmul(A.z, dot)), A.w);
    }
    const double ic = icnt[vid];
    dmi[vid] = make_double4(d[0] * ic, d[1] * ic, d[2] * ic, 0.0);
  }
  block_add_to(local, loss);
}

// pass T2: per-tet chain through the tet normal (_core.pyx:651-667): dL/df per slot and g
// (zeros where the reference skips the tet); one thread per cell, 6 tets
template <int p>
__device__ __forceinline__ void t2_tet(const CellCorners& K, const double4* __restrict__ dmi, float4* __restrict__ tdf,
                                       float4* __restrict__ tg) {
  // FP64 throughout, but with reciprocals instead of the reference's repeated divisions: the
  // results are rounded to FP32 for the gradient buffer anyway (the skip tests are unchanged)
  uint32_t v[4];
  double P[4][3], f[4];
  cell_tet<p>(K, v, P, f);
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
        const double4 m = dmi[v[c]];
        dnt[0] += m.x;
        dnt[1] += m.y;
        dnt[2] += m.z;
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
  *tdf = o;
  *tg = og;
}

__global__ void __launch_bounds__(256) k_nc_tet_chain(int64_t C, int64_t c_lo, int64_t c_hi, Grid G,
                                                      const double* __restrict__ sdf,
                                                      const double* __restrict__ deform,
                                                      const double4* __restrict__ dmi, float4* __restrict__ tdf,
                                                      float4* __restrict__ tg) {
  for (int64_t c = c_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < c_hi;
       c += (int64_t)gridDim.x * blockDim.x) {
    CellCorners K;
    load_cell((uint32_t)c, G, sdf, deform, K);
    t2_tet<0>(K, dmi, tdf + c, tg + c);
    t2_tet<1>(K, dmi, tdf + C + c, tg + C + c);
    t2_tet<2>(K, dmi, tdf + 2 * C + c, tg + 2 * C + c);
    t2_tet<3>(K, dmi, tdf + 3 * C + c, tg + 3 * C + c);
    t2_tet<4>(K, dmi, tdf + 4 * C + c, tg + 4 * C + c);
    t2_tet<5>(K, dmi, tdf + 5 * C + c, tg + 5 * C + c);
  }
}

// pass C: per-vertex gather of the per-tet chain terms
__global__ void __launch_bounds__(256) k_nc_grad(int64_t lo, int64_t hi, Grid G, const float4* __restrict__ tdf,
                                                 const float4* __restrict__ tg, float scale,
                                                 float* __restrict__ d_vert, Fx fx) {
  for (int64_t vid = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vid < hi;
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
    if (fx.vert)
      fx_add4(fx.vert + vid * 4, scale * ds, scale * dp[0], scale * dp[1], scale * dp[2], fx.bad);
    else
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
                                              double b2, double c1, double c2, double eps, double limit,
                                              const float* __restrict__ status) {
  // status (nullable): [0] non-finite map gradients seen by the backward, [1] non-finite
  // gradient entries (k_finite_check), [2] overflowed sync-free views — the update is skipped
  // and the caller raises (or re-runs the step)
  // (raster.py:209-211, fit.py:209-212 check before opt.step)
  if (status && (status[0] != 0.f || status[1] != 0.f || status[2] != 0.f)) return;
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

// count the non-finite entries of the gradient buffer into *flag (warp-aggregated)
__global__ void __launch_bounds__(256) k_finite_check(int64_t n4, const float4* __restrict__ g4, float* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 g = g4[i];
    bad |= !isfinite(g.x) || !isfinite(g.y) || !isfinite(g.z) || !isfinite(g.w);
  }
  if (__ballot_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAdd(flag, 1.0f);
}

// fixed-point gradients (deterministic mode) -> FP32; the dropped-contribution count fx[n]
// goes to status[1] (non-finite gradient entries: Adam skips the step)
__global__ void __launch_bounds__(256) k_fx_to_f32(int64_t n, const long long* __restrict__ fx,
                                                   float* __restrict__ out, float* __restrict__ status) {
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = fx_value(fx[i]);
  if (status && i0 == 0 && fx[n] != 0) atomicAdd(status + 1, (float)fx[n]);
}

}  // namespace ts

using namespace ts;

void ts_impl_fx_to_f32(const long long* fx, int64_t n, float* out, float* status, cudaStream_t st) {
  if (n <= 0) return;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_fx_to_f32<<<blocks, 256, 0, st>>>(n, fx, out, status);
}

void ts_impl_adam(int64_t N, const float* g4, double* sdf, double* deform, double* m_sdf, double* v_sdf,
                  double* m_def, double* v_def, double lr_sdf, double lr_def, double b1, double b2, int64_t t,
                  double eps, double limit, cudaStream_t st, float* status) {
  if (N <= 0) return;
  const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
  int blocks = (int)((N + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (status) k_finite_check<<<blocks, 256, 0, st>>>(N, reinterpret_cast<const float4*>(g4), status + 1);
  k_adam<<<blocks, 256, 0, st>>>(N, reinterpret_cast<const float4*>(g4), sdf, deform, m_sdf, v_sdf, m_def, v_def,
                                 lr_sdf, lr_def, b1, b2, c1, c2, eps, limit, status);
}

void ts_impl_eikonal(const double* sdf, const double* deform, int R, const int32_t* tet_set, int64_t n, float scale,
                     float* d_vert, double* loss, cudaStream_t st, const Fx* fx) {
  cudaMemsetAsync(loss, 0, sizeof(double), st);
  if (n <= 0) return;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_eikonal<<<blocks, 256, 0, st>>>(n, tet_set, make_grid(R), sdf, deform, scale, d_vert, loss, fx ? *fx : Fx{});
}

// scratch layout of the normal-consistency passes (16-byte aligned pieces)
static void nc_layout(int R, int64_t off[8]) {
  const int64_t n = R + 1, N = n * n * n, T = 6 * (int64_t)R * R * R;
  const int64_t sz[7] = {32 * N, 32 * N, 8 * N, 0, 32 * T, 16 * T, 16 * T};  // nv dmi icnt - tn tdf tg
  off[0] = 0;
  for (int i = 0; i < 7; ++i) off[i + 1] = off[i] + ((sz[i] + 255) & ~255ll);
}

int64_t ts_impl_nc_scratch_bytes(int R) {
  int64_t off[8];
  nc_layout(R, off);
  return off[7];
}

// scratch: ts_impl_nc_scratch_bytes(R) bytes of device memory, or nullptr (stream-ordered pool)
// z0 / z1: the vertex layers [z0, z1) whose gradient (and whose edges' penalty) this call adds
// (default all); each pass covers the layers it needs: grad [z0, z1) <- tet chain cells
// [z0 - 1, z1) <- edge terms [z0 - 1, z1 + 1) <- vertex normals [z0 - 2, z1 + 2) <- tet
// normals cells [z0 - 3, z1 + 2), clamped to the grid.
void ts_impl_normal_consistency(const double* sdf, const double* deform, int R, float scale, float* d_vert,
                                double* loss, cudaStream_t st, void* scratch, const Fx* fx, int z0, int z1) {
  const int64_t n = R + 1, N = n * n * n, T = 6 * (int64_t)R * R * R;
  cudaMemsetAsync(loss, 0, sizeof(double), st);
  int64_t off[8];
  nc_layout(R, off);
  char* base = static_cast<char*>(scratch);
  if (!base) cudaMallocAsync(reinterpret_cast<void**>(&base), off[7], st);
  double4* nv = reinterpret_cast<double4*>(base + off[0]);   // A: unit vertex normals, .w = |mean|
  double4* dmi = reinterpret_cast<double4*>(base + off[1]);  // B: edge terms / count
  double* icnt = reinterpret_cast<double*>(base + off[2]);
  double4* tn = reinterpret_cast<double4*>(base + off[4]);   // T1: unit tet normals (FP64: they feed the loss)
  float4* tdf = reinterpret_cast<float4*>(base + off[5]);    // T2: per-tet chain terms (FP32: gradient only)
  float4* tg = reinterpret_cast<float4*>(base + off[6]);
  const Grid G = make_grid(R);
  const int64_t C = T / 6;
  if (z1 < 0 || z1 > n) z1 = (int)n;
  if (z0 < 0) z0 = 0;
  auto vr = [&](int a, int b, int64_t& lo, int64_t& hi) {  // vertex layers [a, b) -> ids
    lo = (int64_t)(a < 0 ? 0 : a) * n * n;
    hi = (int64_t)(b > n ? n : b) * n * n;
  };
  auto cr = [&](int a, int b, int64_t& lo, int64_t& hi) {  // cell layers [a, b) -> ids
    lo = (int64_t)(a < 0 ? 0 : a) * R * R;
    hi = (int64_t)(b > R ? R : b) * R * R;
  };
  auto blocks = [](int64_t a, int64_t b) {
    const int64_t k = (b - a + 255) / 256;
    return (int)(k < 1 ? 1 : (k < 148 * 8 ? k : 148 * 8));
  };
  int64_t tn_lo, tn_hi, nv_lo, nv_hi, e_lo, e_hi, own_lo, own_hi, ch_lo, ch_hi;
  cr(z0 - 3, z1 + 2, tn_lo, tn_hi);
  vr(z0 - 2, z1 + 2, nv_lo, nv_hi);
  vr(z0 - 1, z1 + 1, e_lo, e_hi);
  vr(z0, z1, own_lo, own_hi);
  cr(z0 - 1, z1, ch_lo, ch_hi);
  if (z0 < z1) {
    k_nc_tet_normals<<<blocks(tn_lo, tn_hi), 256, 0, st>>>(C, tn_lo, tn_hi, G, sdf, deform, tn);
    k_nc_vertex_normals<<<blocks(nv_lo, nv_hi), 256, 0, st>>>(nv_lo, nv_hi, G, tn, nv, icnt);
    k_nc_edges<<<blocks(e_lo, e_hi), 256, 0, st>>>(e_lo, e_hi, own_lo, own_hi, G, nv, icnt, dmi, loss);
    k_nc_tet_chain<<<blocks(ch_lo, ch_hi), 256, 0, st>>>(C, ch_lo, ch_hi, G, sdf, deform, dmi, tdf, tg);
    k_nc_grad<<<blocks(own_lo, own_hi), 256, 0, st>>>(own_lo, own_hi, G, tdf, tg, scale, d_vert, fx ? *fx : Fx{});
  }
  (void)N;
  if (!scratch) cudaFreeAsync(base, st);
}
