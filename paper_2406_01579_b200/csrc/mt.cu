// mt.cu — K9 Marching Tetrahedra (grid.py:120-239), bit-exact with the reference.
//
// The reference collects crossing slots per tet, np.unique's them into sorted grid edges,
// interpolates one vertex per edge, emits triangles in the group order
// [1-negative tets][3-negative tets][quad t1 of 2-2 tets][quad t2], orients them along the
// tet gradient, then welds equal positions (np.unique over rows) and drops degenerate
// triangles.  On the implicit Kuhn grid the same result is built without materialising
// connectivity:
//   E1  per vertex a: 7 sign-change flags for its forward Kuhn edges (deltas 1, n, n+1, n^2,
//       n^2+1, n^2+n, n^2+n+1 — ascending, so (a, slot) order IS the lexicographic edge
//       order) -> per-32-vertex-word counts, exclusive scan + in-word popcounts = the index
//       of each crossing edge in np.unique's output; the crossing edges listed in that order
//   E2  crossing positions p = (f_b v_a - f_a v_b) / (f_b - f_a) in FP64 without
//       contraction, endpoint snap on f == 0 (grid.py:120-133), one thread per edge
//   T1  per tet class counts in 2048-tet chunks, scans -> group-ordered output slots (with
//       R % 8 == 0 from z-fastest sign rows: eight cells per four word windows)
//   T2  per crossing tet: slot edges, quad diagonal rule (np.isclose + min-parent key),
//       orientation against the cross-product tet gradient
//   W   weld: merge sort (1024-key shared-memory block sorts, then merge-path passes) of the
//       crossing vertices by (x, y, z) (order-preserving u64 keys,
//       -0 == +0), group ids by adjacent-difference scan, remap, degenerate filter
//       (distinct indices and |cross| > 1e-14, FP64 numpy order) and order-preserving
//       compaction.
// Integer/FP64 stream work, HBM-bound; runs once per extraction.
#include "internal.cuh"
#include "scan.cuh"

#include <initializer_list>

namespace ts {

__device__ __forceinline__ int64_t edge_delta(int s, int64_t n) {
  const int64_t d[7] = {1, n, n + 1, n * n, n * n + 1, n * n + n, n * n + n + 1};
  return d[s];
}
__device__ __forceinline__ void edge_off(int s, int& ox, int& oy, int& oz) {
  ox = (s == 0 || s == 2 || s == 4 || s == 6);
  oy = (s == 1 || s == 2 || s == 5 || s == 6);
  oz = (s >= 3);
}

// E1: per-vertex crossing flags (bit s: the sign differs across forward edge s), negbits = one
// "f < 0" bit per vertex (2 MB at 256^3: the per-cell classification reads it from L2), and the
// crossing-edge count of every 32-vertex word (scanned into per-word bases: a vertex's first
// edge index = its word's base + the flag popcounts of the vertices before it in the word —
// no per-vertex count / offset arrays)
__global__ void k_mt_vflags(int64_t N, Grid G, const double* __restrict__ sdf, uint8_t* __restrict__ flags,
                            int32_t* __restrict__ wcnt, uint32_t* __restrict__ negbits) {
  for (int64_t a0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); a0 < N;
       a0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = a0 + (threadIdx.x & 31);
    bool na = false;
    uint32_t fl = 0;
    if (a < N) {
      int x, y, z;
      vertex_xyz((uint32_t)a, G, x, y, z);
      na = sdf[a] < 0.0;
#pragma unroll
      for (int s = 0; s < 7; ++s) {
        int ox, oy, oz;
        edge_off(s, ox, oy, oz);
        if (x + ox > G.R || y + oy > G.R || z + oz > G.R) continue;
        const int64_t b = a + edge_delta(s, G.n);
        if ((sdf[b] < 0.0) != na) fl |= 1u << s;
      }
      flags[a] = (uint8_t)fl;
    }
    const unsigned w = __ballot_sync(0xffffffffu, na);
    const int c = warp_sum(__popc(fl));
    if ((threadIdx.x & 31) == 0) {
      negbits[a0 >> 5] = w;
      wcnt[a0 >> 5] = c;
    }
  }
}

// E1b: the crossing edges in np.unique order, elist[e] = a << 3 | s — one warp per 32-vertex
// word with crossings (the words' bases from the scan, ranks by a warp scan of the counts)
__global__ void k_mt_elist(int64_t N, const uint8_t* __restrict__ flags, const int64_t* __restrict__ wbase,
                           int64_t* __restrict__ elist) {
  const int64_t nw = (N + 31) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t e0 = __ldg(wbase + w);
    if (__ldg(wbase + w + 1) == e0) continue;  // (warp-uniform)
    const int64_t a = (w << 5) + lane;
    const uint32_t fl = a < N ? flags[a] : 0u;
    const int c = __popc(fl);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int64_t e = e0 + incl - c;
    for (uint32_t m = fl; m; m &= m - 1u) elist[e++] = (a << 3) | (__ffs(m) - 1);
  }
}

// first crossing-edge index of vertex a: its word's base + the flag popcounts of the vertices
// a0 .. a - 1 of the word (flags padded to whole 32-byte words)
__device__ __forceinline__ int64_t vbase(const uint8_t* __restrict__ flags, const int64_t* __restrict__ wbase,
                                         int64_t a) {
  const int r = (int)(a & 31);
  const uint4* f4 = reinterpret_cast<const uint4*>(flags + (a - r));
  const uint4 lo = __ldg(f4), hi = __ldg(f4 + 1);
  const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
  int c = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int nb = r - 4 * k;  // bytes of word k before a
    const uint32_t m = nb >= 4 ? 0xffffffffu : (nb <= 0 ? 0u : (1u << (8 * nb)) - 1u);
    c += __popc(w[k] & m);
  }
  return wbase[a >> 5] + c;
}

__device__ __forceinline__ int64_t edge_index(const uint8_t* flags, const int64_t* ebase, int64_t a, int64_t b,
                                              int64_t n) {
  if (a > b) {
    int64_t t = a;
    a = b;
    b = t;
  }
  const int64_t d = b - a;
  int s = d == 1 ? 0 : d == n ? 1 : d == n + 1 ? 2 : d == n * n ? 3 : d == n * n + 1 ? 4 : d == n * n + n ? 5 : 6;
  return vbase(flags, ebase, a) + __popc((uint32_t)flags[a] & ((1u << s) - 1u));
}

// E2: crossing positions (_edge_crossings, grid.py:120-133), one thread per crossing edge
__global__ void k_mt_verts(int64_t V, Grid G, const double* __restrict__ sdf, const double* __restrict__ deform,
                           const int64_t* __restrict__ elist, double* __restrict__ verts) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < V; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t code = __ldg(elist + e);
    const int64_t a = code >> 3, b = a + edge_delta((int)(code & 7), G.n);
    const double fa = sdf[a], fb = sdf[b];
    double pa[3], pb[3], p[3];
    vertex_position((uint32_t)a, G, deform, pa);
    vertex_position((uint32_t)b, G, deform, pb);
    if (fa == 0.0) {
      p[0] = pa[0]; p[1] = pa[1]; p[2] = pa[2];
    } else if (fb == 0.0) {
      p[0] = pb[0]; p[1] = pb[1]; p[2] = pb[2];
    } else {
      const double den = dsub(fb, fa);
      for (int c = 0; c < 3; ++c) p[c] = ddiv(dsub(dmul(fb, pa[c]), dmul(fa, pb[c])), den);
    }
    verts[e * 3 + 0] = p[0];
    verts[e * 3 + 1] = p[1];
    verts[e * 3 + 2] = p[2];
  }
}

// Crossing tets are classified per CELL: the 8 corner signs form a mask, each tet's class is
// the popcount of (mask & its corner mask) — 1 / 3: one triangle, 2: two.  Cells are taken in
// tet-id order (cell = ix R^2 + iy R + iz; tet = cell * 6 + p), so per-thread cell ranges
// plus block scans give the reference's group-ordered output slots.
constexpr int kCellsPerThread = 8;
constexpr int kCellChunk = kScanThreads * kCellsPerThread;  // cells per CTA

__device__ __forceinline__ uint32_t tet_cmask(int p) {
  return (1u << perm_corner(p, 0)) | (1u << perm_corner(p, 1)) | (1u << perm_corner(p, 2)) | (1u << perm_corner(p, 3));
}

// negative-corner mask of cell c (f < 0 inside, f = 0 counts as outside) from the vertex bits
__device__ __forceinline__ uint32_t cell_negmask(uint32_t c, const Grid& G, const uint32_t* __restrict__ negbits) {
  const uint32_t q = G.dR.div(c);  // ix*R + iy
  const uint32_t iz = c - q * (uint32_t)G.R;
  const uint32_t ix = G.dR.div(q);
  const uint32_t iy = q - ix * (uint32_t)G.R;
  const uint32_t n = (uint32_t)G.n;
  const uint32_t v0 = ix + n * (iy + n * iz);
  uint32_t m = 0;
#pragma unroll
  for (int lc = 0; lc < 8; ++lc) {
    const uint32_t v = v0 + (lc & 1) + n * (((lc >> 1) & 1) + n * ((lc >> 2) & 1));
    m |= ((__ldg(negbits + (v >> 5)) >> (v & 31)) & 1u) << lc;
  }
  return m;
}

// The same signs with z fastest: row (x, y) = ww words holding bit z of vertex (x, y, z),
// z = 0..R (32 x 32 bit blocks of negbits transposed).  With R % 8 == 0 a thread's
// eight cells c0..c0+7 share (ix, iy), so their 4 x 9 corner bits are four shifted row windows
// — two word loads each instead of 64 scattered bit loads — and the eight cells are skipped at
// once when all 36 bits agree (no crossing: almost every cell of the grid).
__global__ void k_mt_zbits(Grid G, const uint32_t* __restrict__ negbits, uint32_t* __restrict__ zbits, int ww) {
  // one warp per (y, 32-x block, 32-z block): lane l takes the 32 x-bits of z = z0 + l (a
  // funnel shift of two words: x rows are not word-aligned), then 32 ballots transpose the
  // 32 x 32 bit block so lane x holds the z word of row (x0 + x, y)
  const int n = G.n, nxb = (n + 31) / 32;
  const int64_t ntask = (int64_t)n * nxb * ww;
  const int lane = threadIdx.x & 31;
  for (int64_t task = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; task < ntask;
       task += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int zb = (int)(task % ww);
    const int64_t rest = task / ww;
    const int xb = (int)(rest % nxb), y = (int)(rest / nxb);
    const int z = zb * 32 + lane;
    uint32_t wl = 0;
    if (z < n) {
      const int64_t v = (int64_t)xb * 32 + (int64_t)n * (y + (int64_t)n * z);
      const int sh = (int)(v & 31);
      const uint32_t lo = __ldg(negbits + (v >> 5)), hi = __ldg(negbits + (v >> 5) + 1);  // (padded)
      wl = sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
    }
    uint32_t out = 0;
#pragma unroll
    for (int x = 0; x < 32; ++x) {
      const unsigned m = __ballot_sync(0xffffffffu, (wl >> x) & 1u);
      if (lane == x) out = m;
    }
    const int xx = xb * 32 + lane;
    if (xx < n) zbits[((int64_t)xx * n + y) * ww + zb] = out;
  }
}

// the 9-bit z windows iz0..iz0+8 of the four corner rows (dx | dy << 1) of cells c0..c0+7
// (c0 % 8 == 0, R % 8 == 0); false when all 36 bits agree
__device__ __forceinline__ bool cell_rows8(uint32_t c0, const Grid& G, const uint32_t* __restrict__ zbits, int ww,
                                           uint32_t (&r)[4]) {
  const uint32_t q = G.dR.div(c0);  // ix*R + iy
  const uint32_t iz0 = c0 - q * (uint32_t)G.R;
  const uint32_t ix = G.dR.div(q);
  const uint32_t iy = q - ix * (uint32_t)G.R;
  const uint32_t n = (uint32_t)G.n, sh = iz0 & 31u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t* p = zbits + (size_t)((ix + (k & 1)) * n + iy + (k >> 1)) * ww + (iz0 >> 5);
    const uint64_t w = (uint64_t)__ldg(p) | (sh > 23u ? (uint64_t)__ldg(p + 1) << 32 : 0ull);
    r[k] = (uint32_t)(w >> sh) & 0x1ffu;
  }
  return (r[0] | r[1] | r[2] | r[3]) != 0u && (r[0] & r[1] & r[2] & r[3]) != 0x1ffu;
}
// negative-corner mask of cell c0 + k from its rows (corner lc = dx | dy << 1 | dz << 2)
__device__ __forceinline__ uint32_t cell_mask8(const uint32_t (&r)[4], int k) {
  uint32_t m = 0;
#pragma unroll
  for (int lc = 0; lc < 8; ++lc) m |= ((r[lc & 3] >> (k + (lc >> 2))) & 1u) << lc;
  return m;
}

// class counts of a cell's 6 tets, packed n1 | n3 << 8 | n2 << 16
__device__ __forceinline__ uint32_t cell_counts(uint32_t m) {
  if (m == 0u || m == 0xffu) return 0u;
  uint32_t r = 0;
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    const int c = __popc(m & tet_cmask(p));
    r += c == 1 ? 1u : (c == 3 ? (1u << 8) : (c == 2 ? (1u << 16) : 0u));
  }
  return r;
}

// T1: per-chunk counts of the three groups
// (zbits != null: the z-fastest rows, R % 8 == 0)
__global__ void __launch_bounds__(kScanThreads) k_mt_ccount(int64_t C, Grid G, const uint32_t* __restrict__ negbits,
                                                           int64_t* __restrict__ c1, int64_t* __restrict__ c3,
                                                           int64_t* __restrict__ c2, const uint32_t* __restrict__ zbits,
                                                           int ww) {
  const int64_t c0 = (int64_t)blockIdx.x * kCellChunk + (int64_t)threadIdx.x * kCellsPerThread;
  uint32_t acc = 0;  // <= 8 cells x 6 tets per field
  if (zbits) {
    uint32_t r[4];
    if (c0 < C && cell_rows8((uint32_t)c0, G, zbits, ww, r))
#pragma unroll
      for (int k = 0; k < kCellsPerThread; ++k) acc += cell_counts(cell_mask8(r, k));
  } else {
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k)
      if (c0 + k < C) acc += cell_counts(cell_negmask((uint32_t)(c0 + k), G, negbits));
  }
  int n1 = warp_sum((int)(acc & 0xffu)), n3 = warp_sum((int)((acc >> 8) & 0xffu)), n2 = warp_sum((int)(acc >> 16));
  __shared__ int s[3][kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = n1;
    s[1][threadIdx.x >> 5] = n3;
    s[2][threadIdx.x >> 5] = n2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0, c = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) a += s[0][w], b += s[1][w], c += s[2][w];
    c1[blockIdx.x] = a;
    c3[blockIdx.x] = b;
    c2[blockIdx.x] = c;
  }
}

// orient triangle tri against the tet gradient g (grid.py:219-225) and store it at `slot`
__device__ __forceinline__ void put_tri(int64_t tri[3], const double g[3], const double* __restrict__ verts,
                                       int64_t slot, int64_t* __restrict__ tris) {
  const double* a0 = verts + tri[0] * 3;
  const double* a1 = verts + tri[1] * 3;
  const double* a2 = verts + tri[2] * 3;
  double u[3], w[3];
  for (int i = 0; i < 3; ++i) {
    u[i] = dsub(a1[i], a0[i]);
    w[i] = dsub(a2[i], a0[i]);
  }
  const double nx_ = dsub(dmul(u[1], w[2]), dmul(u[2], w[1]));
  const double ny_ = dsub(dmul(u[2], w[0]), dmul(u[0], w[2]));
  const double nz_ = dsub(dmul(u[0], w[1]), dmul(u[1], w[0]));
  const double dot = dadd(dadd(dmul(nx_, g[0]), dmul(ny_, g[1])), dmul(nz_, g[2]));
  if (dot < 0.0) {
    const int64_t tmp = tri[1];
    tri[1] = tri[2];
    tri[2] = tmp;
  }
  for (int i = 0; i < 3; ++i) tris[slot * 3 + i] = tri[i];
}

__device__ __forceinline__ void tet_grad_of(uint32_t t, const Grid& G, const double* __restrict__ sdf,
                                            const double* __restrict__ deform, double g[3]) {
  double P[4][3], f[4], cc1[3], cc2[3], cc3[3];
  uint32_t vv[4];
  load_tet(t, G, sdf, deform, vv, P, f);
  tet_gradient(P, f, g, cc1, cc2, cc3);
}

// one triangle of a 1- or 3-negative tet at `slot`
__device__ void emit_single(uint32_t t, int c, int64_t slot, const Grid& G, const double* __restrict__ sdf,
                            const double* __restrict__ deform, const uint8_t* __restrict__ flags,
                            const int64_t* __restrict__ ebase, const double* __restrict__ verts,
                            int64_t* __restrict__ tris) {
  uint32_t v[4];
  tet_vertices(t, G, v);
  bool neg[4];
  for (int i = 0; i < 4; ++i) neg[i] = sdf[v[i]] < 0.0;
  // lone vertex = first vertex of the minority sign; the others in local order
  const bool lone_neg = c == 1;
  int m = 0;
  for (int i = 3; i >= 0; --i)
    if (neg[i] == lone_neg) m = i;
  int64_t tri[3];
  int q = 0;
  for (int i = 0; i < 4; ++i)
    if (i != m) tri[q++] = edge_index(flags, ebase, v[m], v[i], G.n);
  double g[3];
  tet_grad_of(t, G, sdf, deform, g);
  put_tri(tri, g, verts, slot, tris);
}

// the two triangles of a 2-2 tet (quad split by the reference's diagonal rule)
__device__ void emit_quad(uint32_t t, int64_t s1, int64_t s2, const Grid& G, const double* __restrict__ sdf,
                          const double* __restrict__ deform, const uint8_t* __restrict__ flags,
                          const int64_t* __restrict__ ebase, const double* __restrict__ verts,
                          int64_t* __restrict__ tris) {
  const int64_t n = G.n;
  uint32_t v[4];
  tet_vertices(t, G, v);
  bool neg[4];
  for (int i = 0; i < 4; ++i) neg[i] = sdf[v[i]] < 0.0;
  int ord[4], q = 0;
  for (int i = 0; i < 4; ++i)
    if (neg[i]) ord[q++] = i;
  for (int i = 0; i < 4; ++i)
    if (!neg[i]) ord[q++] = i;
  const int64_t I = v[ord[0]], J = v[ord[1]], Kv = v[ord[2]], Lv = v[ord[3]];
  const int64_t ik = edge_index(flags, ebase, I, Kv, n), il = edge_index(flags, ebase, I, Lv, n);
  const int64_t jl = edge_index(flags, ebase, J, Lv, n), jk = edge_index(flags, ebase, J, Kv, n);
  auto dist = [&](int64_t p, int64_t q2) {
    const double* A = verts + p * 3;
    const double* B = verts + q2 * 3;
    double s = 0.0;
    for (int i = 0; i < 3; ++i) {
      const double d = dsub(A[i], B[i]);
      s = dadd(s, dmul(d, d));
    }
    return sqrt(s);
  };
  const double d1 = dist(ik, jl), d2 = dist(il, jk);
  const int64_t key1 = min(min(I, Kv), min(J, Lv)), key2 = min(min(I, Lv), min(J, Kv));
  const bool close = fabs(dsub(d1, d2)) <= dadd(1e-8, dmul(1e-5, fabs(d2)));  // np.isclose
  const bool use1 = close ? (key1 <= key2) : (d1 < d2);
  int64_t T1[3], T2[3];
  if (use1) {
    T1[0] = ik; T1[1] = il; T1[2] = jl;
    T2[0] = ik; T2[1] = jl; T2[2] = jk;
  } else {
    T1[0] = ik; T1[1] = il; T1[2] = jk;
    T2[0] = il; T2[1] = jl; T2[2] = jk;
  }
  double g[3];
  tet_grad_of(t, G, sdf, deform, g);
  put_tri(T1, g, verts, s1, tris);
  put_tri(T2, g, verts, s2, tris);
}

// T2a: the crossing tets in the reference's group order: tlist[pos] = tet id, pos = r1
// (1-negative), n1 + r3 (3-negative), n1 + n3 + r2 (2-2); o1/o3/o2 = exclusive per-chunk
// offsets of the three groups (k_mt_ccount + scans)
__global__ void __launch_bounds__(kScanThreads) k_mt_clist(int64_t C, Grid G, const uint32_t* __restrict__ negbits,
                                                          const int64_t* __restrict__ o1, const int64_t* __restrict__ o3,
                                                          const int64_t* __restrict__ o2, int64_t n1, int64_t n3,
                                                          uint32_t* __restrict__ tlist, const uint32_t* __restrict__ zbits,
                                                          int ww) {
  const int64_t c0 = (int64_t)blockIdx.x * kCellChunk + (int64_t)threadIdx.x * kCellsPerThread;
  uint32_t masks[kCellsPerThread];
  uint32_t acc = 0;
  if (zbits) {
    uint32_t r[4];
    const bool any = c0 < C && cell_rows8((uint32_t)c0, G, zbits, ww, r);
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k) {
      masks[k] = any ? cell_mask8(r, k) : 0u;
      acc += cell_counts(masks[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k) {
      masks[k] = c0 + k < C ? cell_negmask((uint32_t)(c0 + k), G, negbits) : 0u;
      acc += cell_counts(masks[k]);
    }
  }
  // block exclusive scan of the three counts (16-bit fields: <= 12288 per CTA, no carries)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t x = (acc & 0xffu) | (((acc >> 8) & 0xffu) << 16), y = acc >> 16;
  uint32_t ix = x, iy = y;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t tx = __shfl_up_sync(0xffffffffu, ix, o), ty = __shfl_up_sync(0xffffffffu, iy, o);
    if (lane >= o) {
      ix += tx;
      iy += ty;
    }
  }
  __shared__ uint32_t wx[kScanThreads / 32], wy[kScanThreads / 32];
  if (lane == 31) {
    wx[wid] = ix;
    wy[wid] = iy;
  }
  __syncthreads();
  uint32_t bx = 0, by = 0;
  for (int w = 0; w < wid; ++w) bx += wx[w], by += wy[w];
  if (acc == 0u) return;
  const uint32_t ex = bx + ix - x, ey = by + iy - y;
  int64_t p1 = o1[blockIdx.x] + (ex & 0xffffu), p3 = n1 + o3[blockIdx.x] + (ex >> 16),
          p2 = n1 + n3 + o2[blockIdx.x] + ey;
#pragma unroll
  for (int k = 0; k < kCellsPerThread; ++k) {
    const uint32_t m = masks[k];
    if (m == 0u || m == 0xffu) continue;
    const uint32_t t0 = (uint32_t)(c0 + k) * 6u;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int cl = __popc(m & tet_cmask(p));
      if (cl == 1) tlist[p1++] = t0 + p;
      else if (cl == 3) tlist[p3++] = t0 + p;
      else if (cl == 2) tlist[p2++] = t0 + p;
    }
  }
}

// T2b: one thread per crossing tet of the list: its triangle(s) at the group-ordered slots
__global__ void __launch_bounds__(256) k_mt_emit(int64_t ncross, Grid G, const double* __restrict__ sdf,
                                                 const double* __restrict__ deform, const uint8_t* __restrict__ flags,
                                                 const int64_t* __restrict__ ebase, const double* __restrict__ verts,
                                                 const uint32_t* __restrict__ tlist, int64_t n1, int64_t n3,
                                                 int64_t n2, int64_t* __restrict__ tris) {
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < ncross;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = tlist[pos];
    if (pos < n1 + n3) {
      emit_single(t, pos < n1 ? 1 : 3, pos, G, sdf, deform, flags, ebase, verts, tris);
    } else {
      const int64_t rank = pos - n1 - n3;
      emit_quad(t, n1 + n3 + rank, n1 + n3 + n2 + rank, G, sdf, deform, flags, ebase, verts, tris);
    }
  }
}

// ---- weld ------------------------------------------------------------------------------
struct VKey {
  unsigned long long x, y, z;
  unsigned long long idx;
};

__device__ __forceinline__ unsigned long long okey(double v) {
  if (v == 0.0) v = 0.0;  // -0 == +0 (np.unique compares values)
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ bool vless(const VKey& a, const VKey& b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  if (a.z != b.z) return a.z < b.z;
  return a.idx < b.idx;
}
__device__ __forceinline__ bool vsame(const VKey& a, const VKey& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

__global__ void k_mt_keys(int64_t V, int64_t P, const double* __restrict__ verts, VKey* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    VKey k;
    if (i < V) {
      k.x = okey(verts[i * 3]);
      k.y = okey(verts[i * 3 + 1]);
      k.z = okey(verts[i * 3 + 2]);
      k.idx = (unsigned long long)i;
    } else {
      k.x = k.y = k.z = ~0ull;
      k.idx = ~0ull;
    }
    keys[i] = k;
  }
}

constexpr int kLocalSort = 1024;  // keys per block of the shared-memory block sort

// Merge sort of the weld keys (replaces the global bitonic network: O(n log n) traffic in
// log2(P / 1024) merge passes instead of O(n log^2 n) compare-exchange launches).
// Block sort: every 1024-key block ascending in shared memory (bitonic, 512 threads).
__global__ void __launch_bounds__(kLocalSort / 2) k_mt_block_sort(VKey* __restrict__ keys) {
  __shared__ VKey sk[kLocalSort];
  const int64_t b0 = (int64_t)blockIdx.x * kLocalSort;
  for (int i = threadIdx.x; i < kLocalSort; i += blockDim.x) sk[i] = keys[b0 + i];
  __syncthreads();
  for (int kk = 2; kk <= kLocalSort; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      const int t = threadIdx.x;
      const int i = 2 * t - (t & (jj - 1));
      const int l = i + jj;
      const bool asc = (i & kk) == 0 || kk == kLocalSort;
      const VKey a = sk[i], b = sk[l];
      if (vless(b, a) == asc) {
        sk[i] = b;
        sk[l] = a;
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kLocalSort; i += blockDim.x) keys[b0 + i] = sk[i];
}

// outputs per thread of a merge pass: one (256-output CTAs, 4x the CTAs of four per thread:
// the passes are latency-bound, 0.93 vs 1.01-1.04 ms per extraction at 256^3)
constexpr int kMergeItems = 1;
// first i in [max(0, d - w), min(d, w)] with B[d - 1 - i] < A[i] (the merge path's split of
// output diagonal d between runs A and B), by a 32-way search of one warp: each round tests 32
// evenly spaced candidates with independent loads (~4 rounds for a 2^18 run, instead of 18
// dependent loads of a binary search)
__device__ __forceinline__ int64_t warp_merge_path(const VKey* __restrict__ A, const VKey* __restrict__ B, int64_t w,
                                                   int64_t d) {
  int64_t lo = d > w ? d - w : 0, hi = d < w ? d : w;  // the answer is in [lo, hi] (hi: sentinel)
  const int lane = threadIdx.x & 31;
  while (lo < hi) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t i = lo + (int64_t)lane * step;
    const bool p = i >= hi || vless(B[d - 1 - i], A[i]);
    const unsigned m = __ballot_sync(0xffffffffu, p);
    if (m == 0u) {  // all 32 candidates below the split
      lo += 31 * step + 1;
      continue;
    }
    const int f = __ffs(m) - 1;
    if (f == 0) break;  // the split is lo
    hi = min(hi, lo + (int64_t)f * step);
    lo += (int64_t)(f - 1) * step + 1;
  }
  return lo;
}

// One merge pass: runs of `w` sorted keys merged pairwise into `out`.  Each CTA produces
// kMergeTile consecutive outputs: warps 0 / 1 find the split of its first / last diagonal,
// the two input windows are staged in shared memory (coalesced), and every thread merges
// kMergeItems outputs after a merge-path search inside the windows.  Keys are unique (idx
// tie-break).
constexpr int kMergeTile = 256 * kMergeItems;
__global__ void __launch_bounds__(256) k_mt_merge(int64_t P, int64_t w, const VKey* __restrict__ in,
                                                 VKey* __restrict__ out) {
  __shared__ VKey sk[kMergeTile];
  __shared__ int64_t split[2];
  const int64_t o0 = (int64_t)blockIdx.x * kMergeTile;
  const int64_t pair0 = o0 / (2 * w) * (2 * w);  // first key of this run pair (2w % kMergeTile == 0)
  const VKey* A = in + pair0;
  const VKey* B = A + w;
  const int64_t d0 = o0 - pair0;
  const int warp = threadIdx.x >> 5;
  if (warp < 2) {
    const int64_t d = d0 + warp * kMergeTile;
    const int64_t sp = d >= 2 * w ? w : warp_merge_path(A, B, w, d);
    if ((threadIdx.x & 31) == 0) split[warp] = sp;
  }
  __syncthreads();
  const int64_t a0 = split[0], b0 = d0 - a0;
  const int na = (int)(split[1] - a0), nb = kMergeTile - na;
  for (int k = threadIdx.x; k < kMergeTile; k += 256) sk[k] = k < na ? A[a0 + k] : B[b0 + (k - na)];
  __syncthreads();
  const VKey* sa = sk;
  const VKey* sb = sk + na;
  const int dd = threadIdx.x * kMergeItems;
  int lo = dd > nb ? dd - nb : 0, hi = dd < na ? dd : na;
  while (lo < hi) {
    const int i = (lo + hi) >> 1;
    if (vless(sb[dd - 1 - i], sa[i])) hi = i;
    else lo = i + 1;
  }
  int i = lo, j = dd - lo;
#pragma unroll
  for (int k = 0; k < kMergeItems; ++k) {
    const bool takeA = j >= nb || (i < na && vless(sa[i], sb[j]));
    out[o0 + dd + k] = takeA ? sa[i] : sb[j];
    if (takeA) ++i;
    else ++j;
  }
}

__global__ void k_mt_newgroup(int64_t V, const VKey* __restrict__ keys, int32_t* __restrict__ first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    first[i] = (i == 0 || !vsame(keys[i], keys[i - 1])) ? 1 : 0;
}

// gid[i] = inclusive scan(first)[i] - 1; writes remap and the unique positions
__global__ void k_mt_remap(int64_t V, const VKey* __restrict__ keys, const int32_t* __restrict__ first,
                           const int64_t* __restrict__ excl, const double* __restrict__ verts,
                           int64_t* __restrict__ remap, double* __restrict__ upos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = excl[i] + first[i] - 1;
    const int64_t src = (int64_t)keys[i].idx;
    remap[src] = g;
    if (first[i])
      for (int c = 0; c < 3; ++c) upos[g * 3 + c] = verts[src * 3 + c];
  }
}

struct TriKeep {
  const int64_t* tris;
  const int64_t* remap;
  const double* upos;
  int64_t* out;
  __device__ bool pred(int64_t t) const {
    const int64_t a = remap[tris[t * 3]], b = remap[tris[t * 3 + 1]], c = remap[tris[t * 3 + 2]];
    if (a == b || b == c || a == c) return false;
    const double* A = upos + a * 3;
    const double* B = upos + b * 3;
    const double* C = upos + c * 3;
    double u[3], w[3];
    for (int i = 0; i < 3; ++i) {
      u[i] = dsub(B[i], A[i]);
      w[i] = dsub(C[i], A[i]);
    }
    const double x = dsub(dmul(u[1], w[2]), dmul(u[2], w[1]));
    const double y = dsub(dmul(u[2], w[0]), dmul(u[0], w[2]));
    const double z = dsub(dmul(u[0], w[1]), dmul(u[1], w[0]));
    return sqrt(dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z))) > 1e-14;
  }
  __device__ void emit(int64_t t, int64_t pos) const {
    for (int i = 0; i < 3; ++i) out[pos * 3 + i] = remap[tris[t * 3 + i]];
  }
};

inline int grid_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

// ---- host pipeline ------------------------------------------------------------------------
struct MtResult {
  double* verts = nullptr;  // welded vertices f64[nv, 3] (device)
  int64_t* tris = nullptr;  // triangles i64[nt, 3] (device)
  int64_t nv = 0, nt = 0;
  cudaStream_t st = nullptr;
};

// sorted keys end up in *keys (the two buffers are swapped as the passes ping-pong)
static void merge_sort(VKey*& keys, VKey*& tmp, int64_t P, cudaStream_t st) {
  // P is a power of two >= kLocalSort
  k_mt_block_sort<<<(unsigned)(P / kLocalSort), kLocalSort / 2, 0, st>>>(keys);
  for (int64_t w = kLocalSort; w < P; w <<= 1) {
    k_mt_merge<<<(unsigned)(P / kMergeTile), 256, 0, st>>>(P, w, keys, tmp);
    VKey* t = keys;
    keys = tmp;
    tmp = t;
  }
}

static void free_all(std::initializer_list<void*> ps, cudaStream_t st) {
  for (void* p : ps)
    if (p) cudaFreeAsync(p, st);
}

// The whole extraction into device buffers owned by `out` (two host syncs: the sizes, the
// final counts).
static int mt_run(const double* sdf, const double* deform, int R, MtResult& out, cudaStream_t st) {
  const Grid G = make_grid(R);
  const int64_t n = R + 1, N = n * n * n, C = (int64_t)R * R * R;
  out.st = st;
  // E1: crossing edges per vertex -> per-32-vertex-word edge index bases
  const int64_t NW = (N + 31) / 32;
  uint8_t* flags = nullptr;
  int32_t* cnt = nullptr;
  int64_t *ebase = nullptr, *scratch = nullptr;
  cudaMallocAsync(&flags, 32 * NW, st);
  cudaMallocAsync(&cnt, sizeof(int32_t) * NW, st);
  cudaMallocAsync(&ebase, sizeof(int64_t) * (NW + 1), st);
  cudaMallocAsync(&scratch, sizeof(int64_t) * compact_blocks(NW), st);
  uint32_t* negbits = nullptr;
  cudaMallocAsync(&negbits, sizeof(uint32_t) * (NW + 8), st);
  k_mt_vflags<<<grid_blocks(N), 256, 0, st>>>(N, G, sdf, flags, cnt, negbits);
  scan_counts(cnt, NW, ebase, scratch, st);
  // T1: per-chunk group counts over cells, exclusive scans
  const int64_t nb = (C + kCellChunk - 1) / kCellChunk;
  int64_t* off = nullptr;  // o1 | o3 | o2, nb + 1 each
  cudaMallocAsync(&off, sizeof(int64_t) * 3 * (nb + 1), st);
  int64_t *o1 = off, *o3 = off + (nb + 1), *o2 = off + 2 * (nb + 1);
  uint32_t* zbits = nullptr;
  const int ww = (int)((n + 31) / 32);
  if (R % 8 == 0) {
    cudaMallocAsync(&zbits, sizeof(uint32_t) * (size_t)(n * n * ww), st);
    k_mt_zbits<<<grid_blocks(32 * n * ((n + 31) / 32) * ww), 256, 0, st>>>(G, negbits, zbits, ww);
  }
  k_mt_ccount<<<(unsigned)nb, kScanThreads, 0, st>>>(C, G, negbits, o1, o3, o2, zbits, ww);
  k_scan_i64<<<3, 1024, 0, st>>>(o1, nb, nb + 1);  // o1, o3, o2
  int64_t h[4];
  cudaMemcpyAsync(&h[0], ebase + NW, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], o1 + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[2], o3 + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[3], o2 + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(cnt, st);
  cudaStreamSynchronize(st);
  const int64_t V = h[0], n1 = h[1], n3 = h[2], n2 = h[3], F = n1 + n3 + 2 * n2;
  if (V == 0 || F == 0) {
    free_all({flags, ebase, scratch, off, negbits, zbits}, st);
    cudaStreamSynchronize(st);
    return 0;
  }
  // E2 + T2: crossing positions, group-ordered oriented triangles
  double* verts = nullptr;
  int64_t* tris = nullptr;
  cudaMallocAsync(&verts, sizeof(double) * 3 * V, st);
  cudaMallocAsync(&tris, sizeof(int64_t) * 3 * F, st);
  int64_t* elist = nullptr;
  cudaMallocAsync(&elist, sizeof(int64_t) * V, st);
  k_mt_elist<<<grid_blocks(32 * NW), 256, 0, st>>>(N, flags, ebase, elist);
  k_mt_verts<<<grid_blocks(V), 256, 0, st>>>(V, G, sdf, deform, elist, verts);
  uint32_t* tlist = nullptr;
  const int64_t ncross = n1 + n3 + n2;
  cudaMallocAsync(&tlist, sizeof(uint32_t) * ncross, st);
  k_mt_clist<<<(unsigned)nb, kScanThreads, 0, st>>>(C, G, negbits, o1, o3, o2, n1, n3, tlist, zbits, ww);
  k_mt_emit<<<grid_blocks(ncross), 256, 0, st>>>(ncross, G, sdf, deform, flags, ebase, verts, tlist, n1, n3, n2, tris);
  // W: weld equal positions (np.unique over rows: lexicographic), remap, drop degenerates
  int64_t P = kLocalSort;
  while (P < V) P <<= 1;
  VKey *keys = nullptr, *ktmp = nullptr;
  cudaMallocAsync(&keys, sizeof(VKey) * P, st);
  cudaMallocAsync(&ktmp, sizeof(VKey) * P, st);
  k_mt_keys<<<grid_blocks(P), 256, 0, st>>>(V, P, verts, keys);
  merge_sort(keys, ktmp, P, st);
  int32_t* first = nullptr;
  int64_t *excl = nullptr, *remap = nullptr, *scratch2 = nullptr;
  cudaMallocAsync(&first, sizeof(int32_t) * V, st);
  cudaMallocAsync(&excl, sizeof(int64_t) * (V + 1), st);
  cudaMallocAsync(&remap, sizeof(int64_t) * V, st);
  cudaMallocAsync(&scratch2, sizeof(int64_t) * compact_blocks(V > F ? V : F), st);
  cudaMallocAsync(&out.verts, sizeof(double) * 3 * V, st);
  cudaMallocAsync(&out.tris, sizeof(int64_t) * 3 * F, st);
  k_mt_newgroup<<<grid_blocks(V), 256, 0, st>>>(V, keys, first);
  scan_counts(first, V, excl, scratch2, st);
  k_mt_remap<<<grid_blocks(V), 256, 0, st>>>(V, keys, first, excl, verts, remap, out.verts);
  TriKeep tk{tris, remap, out.verts, out.tris};
  int64_t* d_total = compact(F, tk, scratch2, st);
  cudaMemcpyAsync(&h[0], d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], excl + V, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  free_all({flags, ebase, scratch, off, negbits, zbits, elist, tlist, verts, tris, keys, ktmp, first, excl, remap, scratch2}, st);
  cudaStreamSynchronize(st);
  out.nt = h[0];
  out.nv = h[1];
  return 0;
}

}  // namespace ts

using namespace ts;

int ts_impl_mt_run(const double* sdf, const double* deform, int R, void** handle, int64_t* nv, int64_t* nt,
                   cudaStream_t st) {
  MtResult* r = new MtResult();
  const int rc = mt_run(sdf, deform, R, *r, st);
  *nv = r->nv;
  *nt = r->nt;
  *handle = r;
  return rc;
}

// copy the result into caller buffers (host or device: cudaMemcpyDefault)
int ts_impl_mt_fetch(void* handle, double* verts, int64_t* tris) {
  MtResult* r = static_cast<MtResult*>(handle);
  if (r->nv && verts)
    cudaMemcpyAsync(verts, r->verts, sizeof(double) * 3 * r->nv, cudaMemcpyDefault, r->st);
  if (r->nt && tris)
    cudaMemcpyAsync(tris, r->tris, sizeof(int64_t) * 3 * r->nt, cudaMemcpyDefault, r->st);
  cudaStreamSynchronize(r->st);
  return 0;
}

void ts_impl_mt_release(void* handle) {
  MtResult* r = static_cast<MtResult*>(handle);
  if (!r) return;
  free_all({r->verts, r->tris}, r->st);
  delete r;
}

int ts_impl_mt_count(const double* sdf, const double* deform, int R, int64_t* nv, int64_t* nt, cudaStream_t st) {
  void* h = nullptr;
  const int rc = ts_impl_mt_run(sdf, deform, R, &h, nv, nt, st);
  ts_impl_mt_release(h);
  return rc;
}

// vertices / triangles: capacities >= the counts of ts_impl_mt_count.  out_n[0] = final
// triangle count, out_n[1] = welded vertex count.
int ts_impl_mt(const double* sdf, const double* deform, int R, double* out_verts, int64_t* out_tris, int64_t* out_n,
               cudaStream_t st) {
  void* h = nullptr;
  int64_t nv = 0, nt = 0;
  int rc = ts_impl_mt_run(sdf, deform, R, &h, &nv, &nt, st);
  if (!rc) rc = ts_impl_mt_fetch(h, out_verts, out_tris);
  ts_impl_mt_release(h);
  out_n[0] = nt;
  out_n[1] = nv;
  return rc;
}
