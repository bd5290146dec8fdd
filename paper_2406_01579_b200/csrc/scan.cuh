// scan.cuh — order-preserving stream compaction and exclusive scans.
//
// Compaction of a predicate functor F (np.nonzero semantics: output order == input order):
//   compact<F>       : k_count (per-CTA survivor counts) -> k_scan_i64 (one CTA) -> k_emit
//                      (re-evaluates F, ranks survivors with warp ballots) — for cheap
//                      predicates over many items (prefilter, MT classification);
//   compact_state<F> : one pass, one item per thread — the predicate's state feeds the
//                      emission and the output offsets come from a decoupled look-back over
//                      the CTA tiles (scene cull / setup).
// scan_counts (int32 counts -> int64 exclusive offsets, total at [n]) is a single decoupled
// look-back pass.
#pragma once
#include "common.cuh"

namespace ts {

constexpr int kScanThreads = 256;
constexpr int kItemsPerThread = 8;
constexpr int kChunk = kScanThreads * kItemsPerThread;  // 2048 items per CTA

// IPT items per thread: 8 for light predicates, 1 for latency-bound ones (more CTAs in flight)
// ---- decoupled look-back (single-pass scans): per tile one status word, flag << 62 | value --
constexpr unsigned long long kLbAgg = 1ull << 62, kLbPre = 2ull << 62, kLbMask = (1ull << 62) - 1;

// logical tile of this CTA in start order (so every predecessor is resident or done)
__device__ __forceinline__ int lb_tile(unsigned long long* ticket) {
  __shared__ int tile;
  if (threadIdx.x == 0) tile = (int)atomicAdd(ticket, 1ull);
  __syncthreads();
  return tile;
}
// warp 0 (all lanes): publish this tile's aggregate, walk back 32 tiles at a time to the
// nearest inclusive prefix, publish ours; returns the exclusive prefix on every lane
__device__ __forceinline__ long long lb_exclusive(unsigned long long* status, int tile, long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) atomicExch(status, kLbPre | (unsigned long long)agg);
    return 0;
  }
  if (lane == 0) atomicExch(status + tile, kLbAgg | (unsigned long long)agg);
  long long prefix = 0;
  for (int hi = tile - 1;;) {
    const int p = hi - lane;  // lane 0 = nearest predecessor
    const unsigned long long w =
        p >= 0 ? *reinterpret_cast<volatile unsigned long long*>(status + p) : (unsigned long long)(2ull << 62);
    const unsigned long long f = w & ~kLbMask;
    if (__any_sync(0xffffffffu, f == 0)) continue;  // a predecessor has not published yet
    const unsigned pm = __ballot_sync(0xffffffffu, f == kLbPre);
    const int k = pm ? __ffs(pm) - 1 : 31;  // nearest inclusive prefix in the window
    long long v = lane <= k ? (long long)(w & kLbMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (pm) break;
    hi -= 32;
  }
  if (lane == 0) atomicExch(status + tile, kLbPre | (unsigned long long)(prefix + agg));
  return prefix;
}

template <class F, int IPT>
__global__ void __launch_bounds__(kScanThreads) k_count(int64_t n, F f, int64_t* __restrict__ counts) {
  const int64_t base = (int64_t)blockIdx.x * (kScanThreads * IPT);
  int c = 0;
#pragma unroll 4
  for (int k = 0; k < IPT; ++k) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n && f.pred(i)) ++c;
  }
  c = warp_sum(c);
  __shared__ int wsum[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += wsum[w];
    counts[blockIdx.x] = t;
  }
}

// exclusive scan of n int64 values in place, total written to a[n] (one CTA, 1024 threads);
// CTA b scans the array at a + b * stride (several equal-length arrays in one launch)
static __global__ void __launch_bounds__(1024) k_scan_i64(int64_t* __restrict__ a, int64_t n, int64_t stride = 0) {
  a += blockIdx.x * stride;
  __shared__ int64_t wtot[32];
  __shared__ int64_t carry_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += 1024) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < n ? a[i] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wtot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int64_t w = wtot[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      wtot[lane] = wi - w;
    }
    __syncthreads();
    int64_t carry = carry_s;
    int64_t excl = carry + wtot[wid] + incl - v;
    if (i < n) a[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry_s = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) a[n] = carry_s;
}

template <class F, int IPT>
__global__ void __launch_bounds__(kScanThreads) k_emit(int64_t n, F f, const int64_t* __restrict__ offs) {
  const int64_t base = (int64_t)blockIdx.x * (kScanThreads * IPT);
  int64_t run = offs[blockIdx.x];
  __shared__ int wcnt[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < IPT; ++k) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    bool p = i < n && f.pred(i);
    unsigned m = __ballot_sync(0xffffffffu, p);
    if (lane == 0) wcnt[wid] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
      int cw = wcnt[w];
      before += (w < wid) ? cw : 0;
      tot += cw;
    }
    if (p) f.emit(i, run + before + __popc(m & ((1u << lane) - 1u)));
    run += tot;
    __syncthreads();
  }
}

// host-side driver: returns the device pointer holding the survivor total (offs[nb])
template <class F, int IPT = kItemsPerThread>
inline int64_t* compact(int64_t n, const F& f, int64_t* offs_scratch, cudaStream_t st) {
  const int64_t chunk = kScanThreads * IPT, nb = (n + chunk - 1) / chunk;
  if (nb > 0) {
    k_count<F, IPT><<<(unsigned)nb, kScanThreads, 0, st>>>(n, f, offs_scratch);
  }
  k_scan_i64<<<1, 1024, 0, st>>>(offs_scratch, nb);
  if (nb > 0) k_emit<F, IPT><<<(unsigned)nb, kScanThreads, 0, st>>>(n, f, offs_scratch);
  return offs_scratch + nb;
}

// One item per thread, for functors whose predicate computes state the emission reuses
// (F::State, pred(i, State&), emit(i, pos, const State&)): a single pass — the predicate is
// evaluated once and the output offsets come from a decoupled look-back over the tiles.
template <class F>
__global__ void __launch_bounds__(kScanThreads, 3) k_compact_lb(int64_t n, F f, unsigned long long* __restrict__ status,
                                                             unsigned long long* __restrict__ ticket, int64_t nb) {
  __shared__ int wcnt[kScanThreads / 32];
  __shared__ long long pre_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tile = lb_tile(ticket);
  const int64_t i = (int64_t)tile * kScanThreads + threadIdx.x;
  typename F::State st;
  const bool p = i < n && f.pred(i, st);
  const unsigned m = __ballot_sync(0xffffffffu, p);
  if (lane == 0) wcnt[wid] = __popc(m);
  __syncthreads();
  int before = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    before += (w < wid) ? wcnt[w] : 0;
    agg += wcnt[w];
  }
  if (wid == 0) {
    const long long pr = lb_exclusive(status, tile, agg);
    if (lane == 0) pre_s = pr;
  }
  __syncthreads();
  const long long pre = pre_s;
  if (p) f.emit(i, pre + before + __popc(m & ((1u << lane) - 1u)), st);
  // the last tile is the last ticket taken: its slot can carry the total
  if (tile == nb - 1 && threadIdx.x == 0) *reinterpret_cast<long long*>(ticket) = pre + agg;
}

// returns the device pointer holding the survivor total (scratch[nb]); scratch needs
// compact_blocks(n, 1) int64 entries
template <class F>
inline int64_t* compact_state(int64_t n, const F& f, int64_t* scratch, cudaStream_t st) {
  const int64_t nb = (n + kScanThreads - 1) / kScanThreads;
  cudaMemsetAsync(scratch, 0, sizeof(int64_t) * (nb + 1), st);
  if (nb > 0)
    k_compact_lb<F><<<(unsigned)nb, kScanThreads, 0, st>>>(n, f, reinterpret_cast<unsigned long long*>(scratch),
                                                           reinterpret_cast<unsigned long long*>(scratch + nb), nb);
  return scratch + nb;
}

inline int64_t compact_blocks(int64_t n, int ipt = kItemsPerThread) {
  return (n + kScanThreads * ipt - 1) / (kScanThreads * ipt) + 1;
}

// ---- exclusive scan of int32 counts into int64 offsets (out[n] = total) --------------
// single pass: each CTA scans kChunk counts (kItemsPerThread consecutive per thread) and gets
// its offset from a decoupled look-back
static __global__ void __launch_bounds__(kScanThreads) k_scan_lb(const int32_t* __restrict__ in, int64_t n,
                                                               int64_t* __restrict__ out,
                                                               unsigned long long* __restrict__ status,
                                                               unsigned long long* __restrict__ ticket, int64_t nb,
                                                               const int64_t* __restrict__ n_dev,
                                                               const int* __restrict__ ovf) {
  __shared__ int64_t ws[kScanThreads / 32];
  __shared__ long long pre_s;
  const int tile = lb_tile(ticket);
  // n_dev (nullable): the valid count on the device (entries [n_dev, n) count as 0);
  // ovf (nullable): the view overflowed its capacities — nothing to scan
  const int64_t nv = ovf && *ovf ? 0 : (n_dev ? min(n, *n_dev) : n);
  const int64_t my = (int64_t)tile * kChunk + (int64_t)threadIdx.x * kItemsPerThread;
  int32_t v[kItemsPerThread];
  int64_t loc = 0;
#pragma unroll
  for (int k = 0; k < kItemsPerThread; ++k) {
    v[k] = (my + k < nv) ? in[my + k] : 0;
    loc += v[k];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[wid] = incl;
  __syncthreads();
  int64_t wbase = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    wbase += (w < wid) ? ws[w] : 0;
    agg += ws[w];
  }
  if (wid == 0) {
    const long long pr = lb_exclusive(status, tile, agg);
    if (lane == 0) pre_s = pr;
  }
  __syncthreads();
  int64_t run = pre_s + wbase + incl - loc;
#pragma unroll
  for (int k = 0; k < kItemsPerThread; ++k) {
    if (my + k < n) out[my + k] = run;
    run += v[k];
  }
  if (tile == nb - 1 && threadIdx.x == kScanThreads - 1) out[n] = run;
}

// scratch needs compact_blocks(n) int64 entries.  n_dev / ovf (device, nullable): see k_scan_lb;
// out[0, n] is written either way (out[n] = the total).
inline void scan_counts(const int32_t* in, int64_t n, int64_t* out, int64_t* scratch, cudaStream_t st,
                        const int64_t* n_dev = nullptr, const int* ovf = nullptr) {
  const int64_t nb = (n + kChunk - 1) / kChunk;
  if (nb == 0) {
    cudaMemsetAsync(out, 0, sizeof(int64_t), st);
    return;
  }
  cudaMemsetAsync(scratch, 0, sizeof(int64_t) * (nb + 1), st);
  k_scan_lb<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, out, reinterpret_cast<unsigned long long*>(scratch),
                                                   reinterpret_cast<unsigned long long*>(scratch + nb), nb, n_dev,
                                                   ovf);
}

}  // namespace ts
