// bin.cu — K3 tile-overlap count/scan/duplicate, K4 per-tile sort, K5 tile ranges.
//
// Replaces raster.bin_and_sort (raster.py:104-141).  The reference duplicates splats in
// splat order, builds key = tile << 32 | q (q = 32-bit fixed-point mean depth) and does
// one global stable argsort.  Inside one tile that order is exactly "sort by (q, splat
// index)", a total order, so the B200 design never sorts globally:
//   count  : per splat, FP64 tile rect (clip(floor(bbox/16))) + q; atomic per-tile counts
//   scan   : tile counts -> starts[T+1] (== the reference's searchsorted starts, K5)
//   scatter: (q << 32 | k) keys into each tile's segment (arbitrary order)
//   sort   : one CTA per tile sorts its segment in shared memory (bitonic, 64-bit keys)
//            and also emits pos_of (splat -> its list positions, for the deterministic
//            gradient gather) and a flag telling whether mean depth is non-decreasing
//            along the list (then the N_w resorting window is the identity, composite.cu).
// All integer work; HBM/L2-bound.
#include "internal.cuh"
#include "scan.cuh"

namespace ts {


// raster.py:118-121 / 132-134, FP64, numpy order
__device__ __forceinline__ void tile_rect_q(const double* bb, double md, int tiles_x, int tiles_y, double near_,
                                            double far_, int& tx0, int& tx1, int& ty0, int& ty1, uint32_t& q) {
  auto tclip = [](double v, int hi) -> int {
    double t = floor(v / 16.0);
    t = t < 0.0 ? 0.0 : t;
    t = t > (double)hi ? (double)hi : t;
    return (int)t;
  };
  tx0 = tclip(bb[0], tiles_x - 1);
  tx1 = tclip(bb[2], tiles_x - 1);
  ty0 = tclip(bb[1], tiles_y - 1);
  ty1 = tclip(bb[3], tiles_y - 1);
  q = depth_key(md, near_, far_);
}

__global__ void k_bin_count(int64_t K, const double* __restrict__ bbox, const double* __restrict__ md, int tiles_x,
                            int tiles_y, double near_, double far_, BinRec* __restrict__ br,
                            uint32_t* __restrict__ qout, int32_t* __restrict__ splat_cnt,
                            int32_t* __restrict__ tile_cnt, const int64_t* __restrict__ Kdev,
                            const int2* __restrict__ prect, const uint32_t* __restrict__ qbits) {
  // Kdev (nullable): the visible splats on the device; K is then the capacity and the
  // counts of [*Kdev, K) are written as 0 (the scans run over the capacity)
  const int64_t n = Kdev ? min(K, *Kdev) : K;
  // warp-uniform loop so the per-tile counter updates can be aggregated per warp: splats
  // with nearby tet ids are nearby in space and mostly share tiles (one atomic per
  // distinct tile per warp instead of one per (splat, tile) pair)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x; k0 < K; k0 += stride) {
    const int64_t k = k0 + threadIdx.x;
    int tx0 = 0, ty0 = 0, nx = 0, ny = 0;
    if (k >= n && k < K) splat_cnt[k] = 0;
    if (k < n) {
      int tx1, ty1;
      uint32_t q;
      tile_rect_q(bbox + k * 4, md[k], tiles_x, tiles_y, near_, far_, tx0, tx1, ty0, ty1, q);
      nx = tx1 - tx0 + 1;
      ny = ty1 - ty0 + 1;
      if (nx < 0) nx = 0;
      if (ny < 0) ny = 0;
      if (prect) {  // fused path: culled tets and splats left out (records.cuh)
        const int2 pr = __ldg(prect + k);
        if (pr.x == kCulledRect) {
          nx = ny = 0;
        } else if (qbits && rect_empty(pr)) {
          const uint32_t h = qhash(q), h2 = qhash2(q);
          const unsigned long long* mx = qtab_max(qbits);
          if (!((__ldg(qbits + (h >> 5)) >> (h & 31)) & 1u) || __ldg(mx + h2) == __ldg(mx + kQTab + h2)) nx = ny = 0;
        }
      }
      br[k] = BinRec{tx0, ty0, nx, ny};
      qout[k] = q;
      splat_cnt[k] = nx * ny;
    }
    const int cnt = nx * ny;
    const int wmax = __reduce_max_sync(0xffffffffu, cnt);
    for (int i = 0; i < wmax; ++i) {
      const int t = i < cnt ? (ty0 + i / nx) * tiles_x + tx0 + i % nx : -1;
      const unsigned same = __match_any_sync(0xffffffffu, t);
      if (t >= 0 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&tile_cnt[t], __popc(same));
    }
  }
}

__global__ void k_bin_scatter(int64_t K, const BinRec* __restrict__ br, const uint32_t* __restrict__ q, int tiles_x,
                              const int64_t* __restrict__ starts, int32_t* __restrict__ cursor,
                              uint64_t* __restrict__ keys, const int64_t* __restrict__ Kdev,
                              const int* __restrict__ ovf) {
  if (ovf && *ovf) return;
  if (Kdev) K = min(K, *Kdev);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const unsigned lane = threadIdx.x & 31;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x; k0 < K; k0 += stride) {
    const int64_t k = k0 + threadIdx.x;
    BinRec b{0, 0, 0, 0};
    uint64_t key = 0;
    if (k < K) {
      b = br[k];
      key = ((uint64_t)q[k] << 32) | (uint64_t)(uint32_t)k;
    }
    const int cnt = b.nx * b.ny;
    const int wmax = __reduce_max_sync(0xffffffffu, cnt);
    for (int i = 0; i < wmax; ++i) {
      const int t = i < cnt ? (b.ty0 + i / b.nx) * tiles_x + b.tx0 + i % b.nx : -1;
      const unsigned same = __match_any_sync(0xffffffffu, t);
      const int leader = __ffs(same) - 1;
      int base = 0;
      if (t >= 0 && (int)lane == leader) base = atomicAdd(&cursor[t], __popc(same));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (t >= 0) {
        TS_ASSERT(starts[t] + base + __popc(same & ((1u << lane) - 1u)) < starts[t + 1]);
        keys[starts[t] + base + __popc(same & ((1u << lane) - 1u))] = key;
      }
    }
  }
}

template <typename Ptr>
__device__ __forceinline__ void bitonic_sort(Ptr s, int P, int nthreads) {
  // every thread owns compare-exchange pairs (not elements): no idle half per stage
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int c = threadIdx.x; c < (P >> 1); c += nthreads) {
        const int i = ((c & ~(j - 1)) << 1) | (c & (j - 1)), ixj = i | j;
        const uint64_t a = s[i], b = s[ixj];
        const bool asc = (i & k) == 0;
        if ((a > b) == asc) {
          s[i] = b;
          s[ixj] = a;
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ void emit_sorted(uint64_t key, int64_t p, int tile, int tiles_x, const BinRec* br,
                                            const int64_t* splat_off, int32_t* items, int32_t* pos_of,
                                            uint32_t* qsorted) {
  int k = (int)(uint32_t)key;
  items[p] = k;
  if (qsorted) qsorted[p] = (uint32_t)(key >> 32);  // the depth key per position (k_window)
  if (!pos_of) return;  // (the fused view path keeps no pos_of)
  BinRec b = br[k];
  int tx = tile % tiles_x, ty = tile / tiles_x;
  int local = (ty - b.ty0) * b.nx + (tx - b.tx0);
  TS_ASSERT(local >= 0 && splat_off[k] + local < splat_off[k + 1]);
  pos_of[splat_off[k] + local] = (int32_t)p;
}

// sort one tile's list in (dynamic) shared memory and emit items / pos_of / nonmono
template <int THREADS>
__device__ __forceinline__ void sort_tile(uint64_t* s, int& bad, int t, const int64_t* __restrict__ starts,
                                          const uint64_t* __restrict__ keys, int tiles_x,
                                          const BinRec* __restrict__ br, const int64_t* __restrict__ splat_off,
                                          const double* __restrict__ md, int32_t* __restrict__ items,
                                          int32_t* __restrict__ pos_of, uint8_t* __restrict__ nonmono,
                                          uint32_t* __restrict__ qsorted) {
  const int64_t lo = starts[t], L = starts[t + 1] - lo;
  int P = 1;
  while (P < L) P <<= 1;
  for (int i = threadIdx.x; i < P; i += THREADS) s[i] = i < L ? keys[lo + i] : ~0ull;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  bitonic_sort(s, P, THREADS);
  int mybad = 0;
  for (int i = threadIdx.x; i < L; i += THREADS) {
    emit_sorted(s[i], lo + i, t, tiles_x, br, splat_off, items, pos_of, qsorted);
    if (i + 1 < L && md[(uint32_t)s[i]] > md[(uint32_t)s[i + 1]]) mybad = 1;
  }
  if (mybad) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) nonmono[t] = (uint8_t)bad;
}

// Long tiles (2048 < L <= 16384), listed by k_long_tiles: persistent 1024-thread CTAs walk the
// list and sort each tile with a shared-memory LSD radix sort (8-bit digits) on q (four
// passes), then order each run of equal q by splat index in place (runs are short; a tile
// with a run longer than 64 is re-sorted on the full key: ceil(splat bits / 8) passes over
// the splat index, then four over q).  Each
// warp owns a striped slab of E * 32 elements (slot e of lane l at w*32E + e*32 + l, so warp
// order is (e, lane) = position order and the sort is stable); ranks inside a warp come from
// __match_any_sync peers and per-warp digit counters, offsets from a digit-major scan of the
// counters.  O(passes * L) instead of the bitonic O(L log^2 L).
#ifndef TS_SMEM_SORT_CAP
#define TS_SMEM_SORT_CAP 4096
#endif
constexpr int kSmemSortCap = TS_SMEM_SORT_CAP;  // longest list sorted by one 256-thread CTA (<= 16 x 256)
constexpr int kRadixThreads = 1024;
constexpr int kRadixWarps = kRadixThreads / 32;

// qdiff / vdiff: OR of (key XOR first key) over the real keys — a pass whose digit is the same
// for every real key is skipped (a stable pass with one occupied bucket, and the padding
// ~0 keys already last, leaves the order unchanged); tiles span a narrow depth band, so the
// top byte of q rarely varies
__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT, int E>
__device__ __forceinline__ void radix_sort_tile(uint32_t* kq, uint32_t* kv, uint32_t* H, uint32_t* dbase,
                                                int passes_lo, uint32_t qdiff, uint32_t vdiff) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int base = w * 32 * E + lane;
  const unsigned lt = (1u << lane) - 1u;
  for (int pass = 0; pass < passes_lo + 4; ++pass) {
    const bool hi = pass >= passes_lo;
    const int shift = (hi ? pass - passes_lo : pass) * 8;
    if ((((hi ? qdiff : vdiff) >> shift) & 255u) == 0u) continue;  // (CTA-uniform)
    for (int i = threadIdx.x; i < NW * 256; i += NT) H[i] = 0u;
    uint32_t q[E], v[E], rk[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      q[e] = kq[base + e * 32];
      v[e] = kv[base + e * 32];
    }
    __syncthreads();
    uint32_t* Hw = H + w * 256;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t d = ((hi ? q[e] : v[e]) >> shift) & 255u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const uint32_t cur = Hw[d];
      rk[e] = cur + __popc(peers & lt);
      __syncwarp();
      if ((peers & lt) == 0u) Hw[d] = cur + __popc(peers);  // lowest peer updates
      __syncwarp();
    }
    __syncthreads();
    // digit-major exclusive scan of the per-warp counters
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
      uint32_t run = 0;
      for (int ww = 0; ww < NW; ++ww) {
        const uint32_t c = H[ww * 256 + d];
        H[ww * 256 + d] = run;
        run += c;
      }
      dbase[d] = run;
    }
    __syncthreads();
    if (w == 0) {
      uint32_t t8[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        t8[k] = dbase[lane * 8 + k];
        sum += t8[k];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        dbase[lane * 8 + k] = run;
        run += t8[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t d = ((hi ? q[e] : v[e]) >> shift) & 255u;
      const uint32_t dst = dbase[d] + Hw[d] + rk[e];
      kq[dst] = q[e];
      kv[dst] = v[e];
    }
    __syncthreads();
  }
}

// Sort P = NT * E keys (q, splat) held as kq / kv in shared memory (L valid, the rest padded
// with ~0): four radix passes on q, then each run of equal q is ordered by splat index in
// place; a run longer than kMaxRun triggers a re-sort on the full key.  `flag` is a shared
// scratch int.
template <int NT, int MAXE>
__device__ __forceinline__ void radix_sort_keys(uint32_t* kq, uint32_t* kv, uint32_t* H, uint32_t* dbase, int P,
                                                int L, int passes_lo, int& flag, uint32_t qdiff, uint32_t vdiff) {
  constexpr int kMaxRun = 64;
  if (threadIdx.x == 0) flag = 0;
  for (int full = 0; full < 2; ++full) {
    const int plo = full ? passes_lo : 0;
    if (MAXE == 8) {
      if (P == 4 * NT)
        radix_sort_tile<NT, 4>(kq, kv, H, dbase, plo, qdiff, vdiff);
      else
        radix_sort_tile<NT, 8>(kq, kv, H, dbase, plo, qdiff, vdiff);
    } else {  // P = NT * E with E = ceil(L / NT) (>= 3): no power-of-two padding
      switch (P / NT) {
        case 3: radix_sort_tile<NT, 3>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        case 4: radix_sort_tile<NT, 4>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        case 5: radix_sort_tile<NT, 5>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        case 6: radix_sort_tile<NT, 6>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        case 7: radix_sort_tile<NT, 7>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        case 8: radix_sort_tile<NT, 8>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        case 12: radix_sort_tile<NT, 12>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
        default: radix_sort_tile<NT, MAXE>(kq, kv, H, dbase, plo, qdiff, vdiff); break;
      }
    }
    if (full) break;
    for (int i = threadIdx.x; i < L; i += NT) {
      if (i > 0 && kq[i - 1] == kq[i]) continue;  // not a run start
      int e = i + 1;
      while (e < L && kq[e] == kq[i] && e - i <= kMaxRun) ++e;
      if (e - i > kMaxRun) {
        flag = 1;
        continue;
      }
      for (int a = i + 1; a < e; ++a) {  // insertion sort of the run by splat index
        const uint32_t x = kv[a];
        int b = a - 1;
        while (b >= i && kv[b] > x) {
          kv[b + 1] = kv[b];
          --b;
        }
        kv[b + 1] = x;
      }
    }
    __syncthreads();
    if (!flag) break;
  }
}

// one CTA per tile for the tiles with 0 < L <= 512: bitonic in 4 KB of shared memory, few
// registers (several CTAs per SM: most lists are this short once the fused path leaves out the
// never-composited splats)
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_tile_sort_bitonic(int T, const int64_t* __restrict__ starts,
                                                              const uint64_t* __restrict__ keys, int tiles_x,
                                                              const BinRec* __restrict__ br,
                                                              const int64_t* __restrict__ splat_off,
                                                              const double* __restrict__ md,
                                                              int32_t* __restrict__ items,
                                                              int32_t* __restrict__ pos_of,
                                                              uint8_t* __restrict__ nonmono,
                                                              uint32_t* __restrict__ qsorted,
                                                              const int* __restrict__ ovf) {
  __shared__ uint64_t s[512];
  __shared__ int bad;
  const int t = blockIdx.x;
  if (t >= T || (ovf && *ovf)) return;
  const int64_t L = starts[t + 1] - starts[t];
  if (L <= 0 || L > 512) return;
  sort_tile<THREADS>(s, bad, t, starts, keys, tiles_x, br, splat_off, md, items, pos_of, nonmono, qsorted);
}

// one CTA per tile for the tiles with 512 < L <= cap (radix)
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_tile_sort_smem(int T, int64_t cap, int passes_lo,
                                                            const int64_t* __restrict__ starts,
                                                            const uint64_t* __restrict__ keys, int tiles_x,
                                                            const BinRec* __restrict__ br,
                                                            const int64_t* __restrict__ splat_off,
                                                            const double* __restrict__ md,
                                                            int32_t* __restrict__ items, int32_t* __restrict__ pos_of,
                                                            uint8_t* __restrict__ nonmono, uint32_t* __restrict__ qsorted,
                                                            const int* __restrict__ ovf) {
  extern __shared__ uint64_t s[];
  __shared__ int bad, longrun;
  __shared__ unsigned long long kdiff;
  const int t = blockIdx.x;
  if (t >= T || (ovf && *ovf)) return;
  const int64_t lo = starts[t], L = starts[t + 1] - lo;
#ifdef TS_SORT_NOSPLIT
  if (L <= 0 || L > cap) return;
  if (L <= 512) {  // (A/B: short lists here too, at this kernel's occupancy)
    sort_tile<THREADS>(reinterpret_cast<uint64_t*>(s), bad, t, starts, keys, tiles_x, br, splat_off, md, items, pos_of,
                       nonmono, qsorted);
    return;
  }
#else
  if (L <= 512 || L > cap) return;  // (L <= 512: k_tile_sort_bitonic)
#endif
  // longer lists: the radix sort of k_tile_sort_long at THREADS threads (kq / kv alias s)
  uint32_t* kq = reinterpret_cast<uint32_t*>(s);
  uint32_t* kv = kq + cap;
  uint32_t* H = kq + 2 * cap;
  uint32_t* dbase = H + (THREADS / 32) * 256;
  // keys per thread: E = ceil(L / THREADS) (>= 3), rounded up to 12 / 16 above 8 (cap <= 16 THREADS)
  int E = (int)((L + THREADS - 1) / THREADS);
  E = E < 3 ? 3 : (E <= 8 ? E : (E <= 12 ? 12 : 16));
  const int P = E * THREADS;
  const uint64_t k0 = keys[lo];
  uint64_t diff = 0;
  for (int i = threadIdx.x; i < P; i += THREADS) {
    const uint64_t k = i < L ? keys[lo + i] : ~0ull;
    if (i < L) diff |= k ^ k0;
    kq[i] = (uint32_t)(k >> 32);
    kv[i] = (uint32_t)k;
  }
  if (threadIdx.x == 0) {
    bad = 0;
    kdiff = 0;
  }
  __syncthreads();
  diff = warp_or64(diff);
  if ((threadIdx.x & 31) == 0 && diff) atomicOr(&kdiff, (unsigned long long)diff);
  __syncthreads();
  radix_sort_keys<THREADS, 16>(kq, kv, H, dbase, P, (int)L, passes_lo, longrun, (uint32_t)(kdiff >> 32),
                               (uint32_t)kdiff);
  int mybad = 0;
  for (int i = threadIdx.x; i < L; i += THREADS) {
    emit_sorted(((uint64_t)kq[i] << 32) | kv[i], lo + i, t, tiles_x, br, splat_off, items, pos_of, qsorted);
    if (i + 1 < L && md[kv[i]] > md[kv[i + 1]]) mybad = 1;
  }
  if (mybad) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) nonmono[t] = (uint8_t)bad;
}

__global__ void __launch_bounds__(kRadixThreads, 1) k_tile_sort_long(
    const int32_t* __restrict__ tlist, const int64_t* __restrict__ tcount, const int64_t* __restrict__ starts,
    const uint64_t* __restrict__ keys, int tiles_x, const BinRec* __restrict__ br,
    const int64_t* __restrict__ splat_off, const double* __restrict__ md, int32_t* __restrict__ items,
    int32_t* __restrict__ pos_of, uint8_t* __restrict__ nonmono, int cap, int passes_lo,
    uint32_t* __restrict__ qsorted, const int* __restrict__ ovf) {
  if (ovf && *ovf) return;
  extern __shared__ uint32_t sm32[];
  __shared__ int longrun;
  __shared__ unsigned long long kdiff;
  uint32_t* kq = sm32;
  uint32_t* kv = sm32 + cap;
  uint32_t* H = sm32 + 2 * cap;
  uint32_t* dbase = H + kRadixWarps * 256;
  __shared__ int bad;
  const int64_t n = *tcount;
  for (int64_t idx = blockIdx.x; idx < n; idx += gridDim.x) {
    const int t = tlist[idx];
    const int64_t lo = starts[t];
    const int L = (int)(starts[t + 1] - lo);
    // keys per thread: E = ceil(L / 1024) (>= 3), rounded up to 12 / 16 above 8
    int E = (L + kRadixThreads - 1) / kRadixThreads;
    E = E < 3 ? 3 : (E <= 8 ? E : (E <= 12 ? 12 : 16));
    const int P = E * kRadixThreads;
    const uint64_t k0 = keys[lo];
    uint64_t diff = 0;
    for (int i = threadIdx.x; i < P; i += kRadixThreads) {
      const uint64_t k = i < L ? keys[lo + i] : ~0ull;  // padding sorts last
      if (i < L) diff |= k ^ k0;
      kq[i] = (uint32_t)(k >> 32);
      kv[i] = (uint32_t)k;
    }
    if (threadIdx.x == 0) {
      bad = 0;
      kdiff = 0;
    }
    __syncthreads();
    diff = warp_or64(diff);
    if ((threadIdx.x & 31) == 0 && diff) atomicOr(&kdiff, (unsigned long long)diff);
    __syncthreads();
    radix_sort_keys<kRadixThreads, 16>(kq, kv, H, dbase, P, L, passes_lo, longrun, (uint32_t)(kdiff >> 32),
                                       (uint32_t)kdiff);
    int mybad = 0;
    for (int i = threadIdx.x; i < L; i += kRadixThreads) {
      emit_sorted(((uint64_t)kq[i] << 32) | kv[i], lo + i, t, tiles_x, br, splat_off, items, pos_of, qsorted);
      if (i + 1 < L && md[kv[i]] > md[kv[i + 1]]) mybad = 1;
    }
    if (mybad) bad = 1;
    __syncthreads();
    if (threadIdx.x == 0) nonmono[t] = (uint8_t)bad;
  }
}

// tiles with lo_len < L <= cap -> tlist[0, *tcount)
__global__ void k_long_tiles(int T, int64_t lo_len, int64_t cap, const int64_t* __restrict__ starts,
                             int32_t* __restrict__ tlist, int64_t* __restrict__ tcount, const int* __restrict__ ovf) {
  if (ovf && *ovf) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const int64_t L = starts[t + 1] - starts[t];
    if (L > lo_len && L <= cap) tlist[atomicAdd((unsigned long long*)tcount, 1ull)] = t;
  }
}

// oversize tiles: bitonic over a padded copy in global scratch (offset 2*lo, size <= 2L)
__device__ void sort_tile_global(int t, int lo_len, const int64_t* __restrict__ starts,
                                 const uint64_t* __restrict__ keys, int tiles_x, const BinRec* __restrict__ br,
                                 const int64_t* __restrict__ splat_off, const double* __restrict__ md,
                                 uint64_t* __restrict__ scratch, int32_t* __restrict__ items,
                                 int32_t* __restrict__ pos_of, uint8_t* __restrict__ nonmono,
                                 uint32_t* __restrict__ qsorted);

// tlist / tcount (nullable): the tiles to sort, listed by k_long_tiles (sync-free path, a
// persistent grid); else CTA t sorts tile t when it is longer than lo_len
__global__ void __launch_bounds__(1024) k_tile_sort_global(int T, int lo_len, const int64_t* __restrict__ starts,
                                                           const uint64_t* __restrict__ keys, int tiles_x,
                                                           const BinRec* __restrict__ br,
                                                           const int64_t* __restrict__ splat_off,
                                                           const double* __restrict__ md,
                                                           uint64_t* __restrict__ scratch,
                                                           int32_t* __restrict__ items, int32_t* __restrict__ pos_of,
                                                           uint8_t* __restrict__ nonmono, uint32_t* __restrict__ qsorted,
                                                           const int* __restrict__ ovf, const int32_t* __restrict__ tlist,
                                                           const int64_t* __restrict__ tcount) {
  if (ovf && *ovf) return;
  const int64_t ntiles = tlist ? *tcount : (int64_t)T;
  for (int64_t idx = blockIdx.x; idx < ntiles; idx += gridDim.x)
    sort_tile_global(tlist ? tlist[idx] : (int)idx, lo_len, starts, keys, tiles_x, br, splat_off, md, scratch, items,
                     pos_of, nonmono, qsorted);
}

__device__ void sort_tile_global(int t, int lo_len, const int64_t* __restrict__ starts,
                                 const uint64_t* __restrict__ keys, int tiles_x, const BinRec* __restrict__ br,
                                 const int64_t* __restrict__ splat_off, const double* __restrict__ md,
                                 uint64_t* __restrict__ scratch, int32_t* __restrict__ items,
                                 int32_t* __restrict__ pos_of, uint8_t* __restrict__ nonmono,
                                 uint32_t* __restrict__ qsorted) {
  __shared__ int bad;
  const int64_t lo = starts[t], L = starts[t + 1] - lo;
  if (L <= lo_len) return;
  int64_t P = 1;
  while (P < L) P <<= 1;
  uint64_t* s = scratch + 2 * lo;
  for (int64_t i = threadIdx.x; i < P; i += 1024) s[i] = i < L ? keys[lo + i] : ~0ull;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int64_t k = 2; k <= P; k <<= 1)
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t c = threadIdx.x; c < (P >> 1); c += 1024) {
        const int64_t i = ((c & ~(j - 1)) << 1) | (c & (j - 1)), ixj = i | j;
        const uint64_t a = s[i], b = s[ixj];
        const bool asc = (i & k) == 0;
        if ((a > b) == asc) { s[i] = b; s[ixj] = a; }
      }
      __threadfence_block();
      __syncthreads();
    }
  int mybad = 0;
  for (int64_t i = threadIdx.x; i < L; i += 1024) {
    emit_sorted(s[i], lo + i, t, tiles_x, br, splat_off, items, pos_of, qsorted);
    if (i + 1 < L && md[(uint32_t)s[i]] > md[(uint32_t)s[i + 1]]) mybad = 1;
  }
  if (mybad) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) nonmono[t] = (uint8_t)bad;
  __syncthreads();  // `bad` is reused by the next tile of a persistent CTA
}

__global__ void k_max_len(int T, const int64_t* __restrict__ starts, int64_t* __restrict__ out) {
  int64_t m = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    int64_t L = starts[t + 1] - starts[t];
    m = L > m ? L : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    int64_t y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)out, (unsigned long long)m);
}

}  // namespace ts

using namespace ts;


// Phase 1: counts, starts[T+1], splat_off[K+1]; returns M and max tile length (host sync).
// dyn (sync-free): K is the capacity, dyn->K the device count; nothing is copied to the host
// (M = starts[T] and the longest list dev_i64[1] stay on the device).
void ts_impl_bin_count(int64_t K, const double* bbox, const double* md, int tiles_x, int tiles_y, double near_,
                       double far_, const BinWork& w, int64_t* starts, int64_t* splat_off, int64_t* M_out,
                       int64_t* maxL_out, cudaStream_t st, const Dyn* dyn, const int2* prect,
                       const uint32_t* qbits) {
  const int T = tiles_x * tiles_y;
  cudaMemsetAsync(w.tile_cnt, 0, sizeof(int32_t) * T, st);
  cudaMemsetAsync(w.dev_i64, 0, sizeof(int64_t) * 2, st);
  if (K > 0) {
    int blocks = (int)((K + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_bin_count<<<blocks, 256, 0, st>>>(K, bbox, md, tiles_x, tiles_y, near_, far_, w.br, w.q, w.splat_cnt,
                                        w.tile_cnt, dyn ? dyn->K : nullptr, prect, qbits);
  }
  scan_counts(w.tile_cnt, T, starts, w.scratch, st);
  if (splat_off) scan_counts(w.splat_cnt, K, splat_off, w.scratch, st);  // (pos_of's offsets; API path)
  k_max_len<<<8, 256, 0, st>>>(T, starts, w.dev_i64 + 1);
  if (dyn) return;
  int64_t h[2];
  cudaMemcpyAsync(&h[0], starts + T, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], w.dev_i64 + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  *M_out = h[0];
  *maxL_out = h[1];
}

// Phase 2: scatter keys + per-tile sort.  keys: [M]; gscratch: [2M] only when maxL > 16384.
// dyn (sync-free): maxL is unknown on the host, so every sort launch runs and picks its tiles
// on the device (bitonic / radix <= 2048 in k_tile_sort_smem, 2048 < L <= 8192 and
// 8192 < L <= 16384 in k_tile_sort_long at two shared-memory sizes, longer in
// k_tile_sort_global, which then needs gscratch [2 * M capacity]); dyn->ovf stops them all.
void ts_impl_bin_sort(int64_t K, int tiles_x, int tiles_y, const double* md, const BinWork& w, const int64_t* starts,
                      const int64_t* splat_off, int64_t maxL, uint64_t* keys, uint64_t* gscratch, int32_t* items,
                      int32_t* pos_of, uint8_t* nonmono, cudaStream_t st, uint32_t* qsorted, const Dyn* dyn) {
  const int T = tiles_x * tiles_y;
  const int* ovf = dyn ? dyn->ovf : nullptr;
  cudaMemsetAsync(w.tile_cnt, 0, sizeof(int32_t) * T, st);
  cudaMemsetAsync(nonmono, 0, T, st);
  if (K > 0) {
    int blocks = (int)((K + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_bin_scatter<<<blocks, 256, 0, st>>>(K, w.br, w.q, tiles_x, starts, w.tile_cnt, keys, dyn ? dyn->K : nullptr,
                                          ovf);
  }
  // sync-free: maxL is the capacity of the longest list (the view overflows above it): the
  // size classes up to it are launched, each picking its tiles on the device
  if (maxL >= 1) {
    int kbits = 1;  // digit passes over the splat index of a full-key sort: ceil(bits(K - 1) / 8)
    while (kbits < 32 && ((int64_t)1 << kbits) < K) ++kbits;
    // lists up to kSmemSortCap: one 256-thread CTA each (bitonic <= 512, radix above; several CTAs
    // per SM), longer ones by the 1024-thread persistent k_tile_sort_long
    const size_t smem_s = sizeof(uint32_t) * (2 * kSmemSortCap + 8 * 256 + 256);  // kq, kv | bitonic u64; H; dbase
    static const bool attr_s = [] {
      cudaFuncSetAttribute(k_tile_sort_smem<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(uint32_t) * (2 * kSmemSortCap + 8 * 256 + 256)));
      return true;
    }();
    (void)attr_s;
#ifndef TS_SORT_NOSPLIT
    k_tile_sort_bitonic<256><<<T, 256, 0, st>>>(T, starts, keys, tiles_x, w.br, splat_off, md, items, pos_of, nonmono,
                                                qsorted, ovf);
    if (dyn || maxL > 512)
#endif
      k_tile_sort_smem<256><<<T, 256, smem_s, st>>>(T, kSmemSortCap, (kbits + 7) / 8, starts, keys, tiles_x, w.br,
                                                    splat_off, md, items, pos_of, nonmono, qsorted, ovf);
    // the attribute is set once, to the 16384-entry cap (a thread-safe static: views in
    // flight launch from several host threads); the launch asks for what it needs
    static const bool attr = [] {
      const size_t mx = sizeof(uint32_t) * (2 * (size_t)16384 + kRadixWarps * 256 + 256);
      cudaFuncSetAttribute(k_tile_sort_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
      return true;
    }();
    (void)attr;
    auto long_sort = [&](int64_t lo_len, int cap) {
      // the scatter cursor is free again: reuse it as the long-tile list
      cudaMemsetAsync(w.dev_i64, 0, sizeof(int64_t), st);
      k_long_tiles<<<(T + 255) / 256, 256, 0, st>>>(T, lo_len, cap, starts, w.tile_cnt, w.dev_i64, ovf);
      const size_t smem = sizeof(uint32_t) * (2 * (size_t)cap + kRadixWarps * 256 + 256);
      const int per_sm = smem <= 110 * 1024 ? 2 : 1;
      k_tile_sort_long<<<148 * per_sm, kRadixThreads, smem, st>>>(w.tile_cnt, w.dev_i64, starts, keys, tiles_x, w.br,
                                                                 splat_off, md, items, pos_of, nonmono, cap,
                                                                 (kbits + 7) / 8, qsorted, ovf);
    };
    if (dyn) {
      if (maxL > kSmemSortCap) long_sort(kSmemSortCap, 8192);
      if (maxL > 8192) long_sort(8192, 16384);
    } else if (maxL > kSmemSortCap) {
      // shared memory sized to the longest list (not the 16384 cap) so two CTAs fit per SM
      // where they can; digit passes over the splat index: ceil(bits(K - 1) / 8)
      long_sort(kSmemSortCap, maxL <= 4096 ? 4096 : (maxL <= 8192 ? 8192 : 16384));
    }
    if (dyn && maxL > 16384) {  // tiles longer than 16384, listed on the device, one persistent CTA per SM
      cudaMemsetAsync(w.dev_i64, 0, sizeof(int64_t), st);
      k_long_tiles<<<(T + 255) / 256, 256, 0, st>>>(T, 16384, (int64_t)1 << 62, starts, w.tile_cnt, w.dev_i64, ovf);
      k_tile_sort_global<<<148, 1024, 0, st>>>(T, 16384, starts, keys, tiles_x, w.br, splat_off, md, gscratch, items,
                                               pos_of, nonmono, qsorted, ovf, w.tile_cnt, w.dev_i64);
    } else if (maxL > 16384) {
      k_tile_sort_global<<<T, 1024, 0, st>>>(T, 16384, starts, keys, tiles_x, w.br, splat_off, md, gscratch, items,
                                             pos_of, nonmono, qsorted, ovf, nullptr, nullptr);
    }
  }
}
