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
//       order) -> exclusive scan = the index of each crossing edge in np.unique's output
//   E2  crossing positions p = (f_b v_a - f_a v_b) / (f_b - f_a) in FP64 without
//       contraction, endpoint snap on f == 0 (grid.py:120-133)
//   T1  per tet class counts in 2048-tet chunks, scans -> group-ordered output slots
//   T2  per crossing tet: slot edges, quad diagonal rule (np.isclose + min-parent key),
//       orientation against the cross-product tet gradient
//   W   weld: bitonic sort of the crossing vertices by (x, y, z) (order-preserving u64 keys,
//       -0 == +0), group ids by adjacent-difference scan, remap, degenerate filter
//       (distinct indices and |cross| > 1e-14, FP64 numpy order) and order-preserving
//       compaction.
// Integer/FP64 stream work, HBM-bound; runs once per extraction.
#include "internal.cuh"
#include "scan.cuh"

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

// E1: per-vertex crossing flags (bit s) and counts
__global__ void k_mt_vflags(int64_t N, Grid G, const double* __restrict__ sdf, uint8_t* __restrict__ flags,
                            int32_t* __restrict__ cnt) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < N; a += (int64_t)gridDim.x * blockDim.x) {
    int x, y, z;
    vertex_xyz((uint32_t)a, G, x, y, z);
    const bool na = sdf[a] < 0.0;
    uint32_t fl = 0;
    for (int s = 0; s < 7; ++s) {
      int ox, oy, oz;
      edge_off(s, ox, oy, oz);
      if (x + ox > G.R || y + oy > G.R || z + oz > G.R) continue;
      const int64_t b = a + edge_delta(s, G.n);
      if ((sdf[b] < 0.0) != na) fl |= 1u << s;
    }
    flags[a] = (uint8_t)fl;
    cnt[a] = __popc(fl);
  }
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
  return ebase[a] + __popc((uint32_t)flags[a] & ((1u << s) - 1u));
}

// E2: crossing positions (_edge_crossings, grid.py:120-133)
__global__ void k_mt_verts(int64_t N, Grid G, const double* __restrict__ sdf, const double* __restrict__ deform,
                           const uint8_t* __restrict__ flags, const int64_t* __restrict__ ebase,
                           double* __restrict__ verts) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < N; a += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t fl = flags[a];
    if (!fl) continue;
    double pa[3], pb[3];
    vertex_position((uint32_t)a, G, deform, pa);
    const double fa = sdf[a];
    int64_t e = ebase[a];
    for (int s = 0; s < 7; ++s) {
      if (!((fl >> s) & 1u)) continue;
      const int64_t b = a + edge_delta(s, G.n);
      vertex_position((uint32_t)b, G, deform, pb);
      const double fb = sdf[b];
      double p[3];
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
      ++e;
    }
  }
}

__device__ __forceinline__ int tet_class(uint32_t t, const Grid& G, const double* __restrict__ sdf) {
  uint32_t v[4];
  tet_vertices(t, G, v);
  int c = 0;
  for (int i = 0; i < 4; ++i) c += sdf[v[i]] < 0.0;
  return c;  // 1, 3: one triangle; 2: two
}

// T1: per-chunk counts of the three groups
__global__ void __launch_bounds__(kScanThreads) k_mt_tcount(int64_t K, Grid G, const double* __restrict__ sdf,
                                                           int64_t* __restrict__ c1, int64_t* __restrict__ c3,
                                                           int64_t* __restrict__ c2) {
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  int n1 = 0, n3 = 0, n2 = 0;
  for (int k = 0; k < kItemsPerThread; ++k) {
    const int64_t t = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (t >= K) break;
    const int c = tet_class((uint32_t)t, G, sdf);
    n1 += c == 1;
    n3 += c == 3;
    n2 += c == 2;
  }
  n1 = warp_sum(n1);
  n3 = warp_sum(n3);
  n2 = warp_sum(n2);
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

// T2: triangles of the crossing tets at their group-ordered slots
__global__ void __launch_bounds__(kScanThreads) k_mt_temit(int64_t K, Grid G, const double* __restrict__ sdf,
                                                          const double* __restrict__ deform,
                                                          const uint8_t* __restrict__ flags,
                                                          const int64_t* __restrict__ ebase,
                                                          const double* __restrict__ verts,
                                                          const int64_t* __restrict__ o1, const int64_t* __restrict__ o3,
                                                          const int64_t* __restrict__ o2, int64_t n1, int64_t n3,
                                                          int64_t n2, int64_t* __restrict__ tris) {
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  int64_t r1 = o1[blockIdx.x], r3 = o3[blockIdx.x], r2 = o2[blockIdx.x];
  __shared__ int wc[3][kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t n = G.n;
  for (int kk = 0; kk < kItemsPerThread; ++kk) {
    const int64_t t = base + (int64_t)kk * kScanThreads + threadIdx.x;
    uint32_t v[4] = {0, 0, 0, 0};
    bool neg[4] = {false, false, false, false};
    int c = 0;
    if (t < K) {
      tet_vertices((uint32_t)t, G, v);
      for (int i = 0; i < 4; ++i) {
        neg[i] = sdf[v[i]] < 0.0;
        c += neg[i];
      }
    }
    const unsigned m1 = __ballot_sync(0xffffffffu, t < K && c == 1);
    const unsigned m3 = __ballot_sync(0xffffffffu, t < K && c == 3);
    const unsigned m2 = __ballot_sync(0xffffffffu, t < K && c == 2);
    if (lane == 0) {
      wc[0][wid] = __popc(m1);
      wc[1][wid] = __popc(m3);
      wc[2][wid] = __popc(m2);
    }
    __syncthreads();
    int b1 = 0, b3 = 0, b2 = 0, t1 = 0, t3 = 0, t2 = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) {
      if (w < wid) b1 += wc[0][w], b3 += wc[1][w], b2 += wc[2][w];
      t1 += wc[0][w], t3 += wc[1][w], t2 += wc[2][w];
    }
    const unsigned lt = (1u << lane) - 1u;
    if (t < K && (c == 1 || c == 3)) {
      // lone vertex = first vertex of the minority sign; the others in local order
      const bool lone_neg = c == 1;
      int m = 0;
      for (int i = 3; i >= 0; --i)
        if (neg[i] == lone_neg) m = i;
      int64_t e[3];
      int q = 0;
      for (int i = 0; i < 4; ++i)
        if (i != m) e[q++] = edge_index(flags, ebase, v[m], v[i], n);
      const int64_t slot = c == 1 ? (r1 + b1 + __popc(m1 & lt)) : (n1 + r3 + b3 + __popc(m3 & lt));
      int64_t tri[3] = {e[0], e[1], e[2]};
      // orientation against the tet gradient (grid.py:219-225)
      double P[4][3], f[4], g[3], cc1[3], cc2[3], cc3[3];
      int xyz[4][3];
      uint32_t vv[4];
      tet_corners((uint32_t)t, G, xyz, vv);
      for (int i = 0; i < 4; ++i) {
        vertex_pos_xyz(xyz[i], vv[i], G, deform, P[i]);
        f[i] = sdf[vv[i]];
      }
      tet_gradient(P, f, g, cc1, cc2, cc3);
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
    } else if (t < K && c == 2) {
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
      const bool close = fabs(dsub(d1, d2)) <= dadd(1e-8, dmul(1e-5, fabs(d2)));
      const bool use1 = close ? (key1 <= key2) : (d1 < d2);
      int64_t T1[3], T2[3];
      if (use1) {
        T1[0] = ik; T1[1] = il; T1[2] = jl;
        T2[0] = ik; T2[1] = jl; T2[2] = jk;
      } else {
        T1[0] = ik; T1[1] = il; T1[2] = jk;
        T2[0] = il; T2[1] = jl; T2[2] = jk;
      }
      const int64_t rank = r2 + b2 + __popc(m2 & lt);
      const int64_t s1 = n1 + n3 + rank, s2 = n1 + n3 + n2 + rank;
      double P[4][3], f[4], g[3], cc1[3], cc2[3], cc3[3];
      int xyz[4][3];
      uint32_t vv[4];
      tet_corners((uint32_t)t, G, xyz, vv);
      for (int i = 0; i < 4; ++i) {
        vertex_pos_xyz(xyz[i], vv[i], G, deform, P[i]);
        f[i] = sdf[vv[i]];
      }
      tet_gradient(P, f, g, cc1, cc2, cc3);
      for (int h = 0; h < 2; ++h) {
        int64_t* tri = h == 0 ? T1 : T2;
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
        const int64_t slot = h == 0 ? s1 : s2;
        for (int i = 0; i < 3; ++i) tris[slot * 3 + i] = tri[i];
      }
    }
    r1 += t1;
    r3 += t3;
    r2 += t2;
    __syncthreads();
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

__global__ void k_mt_bitonic(int64_t P, int64_t kk, int64_t jj, VKey* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i ^ jj;
    if (l <= i) continue;
    const VKey a = keys[i], b = keys[l];
    const bool asc = (i & kk) == 0;
    if (vless(b, a) == asc) {
      keys[i] = b;
      keys[l] = a;
    }
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

struct MtCounts {
  int64_t V, n1, n3, n2;
};

// shared first half: vertex flags + edge bases + triangle group counts
static int mt_counts(const double* sdf, int R, uint8_t** flags, int64_t** ebase, MtCounts& mc, int64_t** o1,
                     int64_t** o3, int64_t** o2, int64_t& nb, cudaStream_t st) {
  const Grid G = make_grid(R);
  const int64_t n = R + 1, N = n * n * n, K = 6ll * R * R * R;
  int32_t* cnt = nullptr;
  int64_t* scratch = nullptr;
  cudaMallocAsync(flags, N, st);
  cudaMallocAsync(&cnt, sizeof(int32_t) * N, st);
  cudaMallocAsync(ebase, sizeof(int64_t) * (N + 1), st);
  cudaMallocAsync(&scratch, sizeof(int64_t) * compact_blocks(N), st);
  k_mt_vflags<<<grid_blocks(N), 256, 0, st>>>(N, G, sdf, *flags, cnt);
  scan_counts(cnt, N, *ebase, scratch, st);
  nb = (K + kChunk - 1) / kChunk;
  cudaMallocAsync(o1, sizeof(int64_t) * (nb + 1), st);
  cudaMallocAsync(o3, sizeof(int64_t) * (nb + 1), st);
  cudaMallocAsync(o2, sizeof(int64_t) * (nb + 1), st);
  k_mt_tcount<<<(unsigned)nb, kScanThreads, 0, st>>>(K, G, sdf, *o1, *o3, *o2);
  k_scan_i64<<<1, 1024, 0, st>>>(*o1, nb);
  k_scan_i64<<<1, 1024, 0, st>>>(*o3, nb);
  k_scan_i64<<<1, 1024, 0, st>>>(*o2, nb);
  int64_t h[4];
  cudaMemcpyAsync(&h[0], *ebase + N, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], *o1 + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[2], *o3 + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[3], *o2 + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(scratch, st);
  cudaStreamSynchronize(st);
  mc = MtCounts{h[0], h[1], h[2], h[3]};
  return 0;
}

}  // namespace ts

using namespace ts;

int ts_impl_mt_count(const double* sdf, const double* deform, int R, int64_t* nv, int64_t* nt, cudaStream_t st) {
  (void)deform;
  uint8_t* flags;
  int64_t *ebase, *o1, *o3, *o2, nb;
  MtCounts mc;
  mt_counts(sdf, R, &flags, &ebase, mc, &o1, &o3, &o2, nb, st);
  *nv = mc.V;
  *nt = mc.n1 + mc.n3 + 2 * mc.n2;
  cudaFreeAsync(flags, st);
  cudaFreeAsync(ebase, st);
  cudaFreeAsync(o1, st);
  cudaFreeAsync(o3, st);
  cudaFreeAsync(o2, st);
  return 0;
}

// vertices: capacity >= count's nv (welded count returned through the first row count);
// triangles: capacity >= count's nt.  *out_nt = final triangle count; the welded vertex
// count is returned as the return value's companion via out_nt[1] when non-null.
int ts_impl_mt(const double* sdf, const double* deform, int R, double* out_verts, int64_t* out_tris, int64_t* out_n,
               cudaStream_t st) {
  const Grid G = make_grid(R);
  const int64_t n = R + 1, N = n * n * n, K = 6ll * R * R * R;
  uint8_t* flags;
  int64_t *ebase, *o1, *o3, *o2, nb;
  MtCounts mc;
  mt_counts(sdf, R, &flags, &ebase, mc, &o1, &o3, &o2, nb, st);
  const int64_t V = mc.V, F = mc.n1 + mc.n3 + 2 * mc.n2;
  if (V == 0 || F == 0) {
    out_n[0] = 0;
    out_n[1] = 0;
    cudaFreeAsync(flags, st);
    cudaFreeAsync(ebase, st);
    cudaFreeAsync(o1, st);
    cudaFreeAsync(o3, st);
    cudaFreeAsync(o2, st);
    cudaStreamSynchronize(st);
    return 0;
  }
  double* verts;
  int64_t* tris;
  cudaMallocAsync(&verts, sizeof(double) * 3 * V, st);
  cudaMallocAsync(&tris, sizeof(int64_t) * 3 * F, st);
  k_mt_verts<<<grid_blocks(N), 256, 0, st>>>(N, G, sdf, deform, flags, ebase, verts);
  k_mt_temit<<<(unsigned)nb, kScanThreads, 0, st>>>(K, G, sdf, deform, flags, ebase, verts, o1, o3, o2, mc.n1, mc.n3,
                                                    mc.n2, tris);
  // weld
  int64_t P = 1;
  while (P < V) P <<= 1;
  VKey* keys;
  cudaMallocAsync(&keys, sizeof(VKey) * P, st);
  k_mt_keys<<<grid_blocks(P), 256, 0, st>>>(V, P, verts, keys);
  for (int64_t kk = 2; kk <= P; kk <<= 1)
    for (int64_t jj = kk >> 1; jj > 0; jj >>= 1) k_mt_bitonic<<<grid_blocks(P), 256, 0, st>>>(P, kk, jj, keys);
  int32_t* first;
  int64_t *excl, *remap, *scratch;
  cudaMallocAsync(&first, sizeof(int32_t) * V, st);
  cudaMallocAsync(&excl, sizeof(int64_t) * (V + 1), st);
  cudaMallocAsync(&remap, sizeof(int64_t) * V, st);
  cudaMallocAsync(&scratch, sizeof(int64_t) * compact_blocks(V > F ? V : F), st);
  k_mt_newgroup<<<grid_blocks(V), 256, 0, st>>>(V, keys, first);
  scan_counts(first, V, excl, scratch, st);
  k_mt_remap<<<grid_blocks(V), 256, 0, st>>>(V, keys, first, excl, verts, remap, out_verts);
  TriKeep tk{tris, remap, out_verts, out_tris};
  int64_t* d_total = compact(F, tk, scratch, st);
  int64_t h[2];
  cudaMemcpyAsync(&h[0], d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], excl + V, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  out_n[0] = h[0];
  out_n[1] = h[1];
  for (void* p : {(void*)flags, (void*)ebase, (void*)o1, (void*)o3, (void*)o2, (void*)verts, (void*)tris,
                  (void*)keys, (void*)first, (void*)excl, (void*)remap, (void*)scratch})
    cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  return 0;
}
