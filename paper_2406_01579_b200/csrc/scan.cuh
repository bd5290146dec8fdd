// scan.cuh — order-preserving stream compaction and exclusive scans.
//
// Compaction is two passes over a predicate functor F:
//   k_count : each CTA owns a contiguous chunk of kChunk items and writes its survivor count
//   k_scan  : one CTA turns the counts into exclusive offsets (+ total at [nb])
//   k_emit  : each CTA re-evaluates F on its chunk, ranks survivors with warp ballots and
//             calls F.emit(i, pos) so output order == input order (np.nonzero semantics)
// Recomputing the predicate is cheaper than materialising flags for the HBM-bound
// predicates used here (prefilter, cull, MT classification).
#pragma once
#include "common.cuh"

namespace ts {

constexpr int kScanThreads = 256;
constexpr int kItemsPerThread = 8;
constexpr int kChunk = kScanThreads * kItemsPerThread;  // 2048 items per CTA

// IPT items per thread: 8 for light predicates, 1 for latency-bound ones (more CTAs in flight)
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

// exclusive scan of n int64 values in place, total written to a[n] (one CTA, 1024 threads)
static __global__ void __launch_bounds__(1024) k_scan_i64(int64_t* __restrict__ a, int64_t n) {
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
// (F::State, pred(i, State&), emit(i, pos, const State&)): the emit pass evaluates once.
template <class F>
__global__ void __launch_bounds__(kScanThreads) k_emit_state(int64_t n, F f, const int64_t* __restrict__ offs) {
  __shared__ int wcnt[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kScanThreads + threadIdx.x;
  typename F::State st;
  const bool p = i < n && f.pred(i, st);
  const unsigned m = __ballot_sync(0xffffffffu, p);
  if (lane == 0) wcnt[wid] = __popc(m);
  __syncthreads();
  int before = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) before += (w < wid) ? wcnt[w] : 0;
  if (p) f.emit(i, offs[blockIdx.x] + before + __popc(m & ((1u << lane) - 1u)), st);
}

template <class F>
inline int64_t* compact_state(int64_t n, const F& f, int64_t* offs_scratch, cudaStream_t st) {
  const int64_t nb = (n + kScanThreads - 1) / kScanThreads;
  if (nb > 0) k_count<F, 1><<<(unsigned)nb, kScanThreads, 0, st>>>(n, f, offs_scratch);
  k_scan_i64<<<1, 1024, 0, st>>>(offs_scratch, nb);
  if (nb > 0) k_emit_state<F><<<(unsigned)nb, kScanThreads, 0, st>>>(n, f, offs_scratch);
  return offs_scratch + nb;
}

inline int64_t compact_blocks(int64_t n, int ipt = kItemsPerThread) {
  return (n + kScanThreads * ipt - 1) / (kScanThreads * ipt) + 1;
}

// ---- exclusive scan of int32 counts into int64 offsets (out[n] = total) --------------
static __global__ void __launch_bounds__(kScanThreads) k_chunk_sums(const int32_t* __restrict__ in, int64_t n,
                                                                  int64_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  int64_t c = 0;
  for (int k = 0; k < kItemsPerThread; ++k) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) c += in[i];
  }
  c = warp_sum(c);
  __shared__ int64_t ws[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

static __global__ void __launch_bounds__(kScanThreads) k_chunk_scan(const int32_t* __restrict__ in, int64_t n,
                                                                  const int64_t* __restrict__ sums,
                                                                  int64_t* __restrict__ out) {
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  // each thread owns kItemsPerThread consecutive items
  const int64_t my = base + (int64_t)threadIdx.x * kItemsPerThread;
  int32_t v[kItemsPerThread];
  int64_t loc = 0;
#pragma unroll
  for (int k = 0; k < kItemsPerThread; ++k) {
    v[k] = (my + k < n) ? in[my + k] : 0;
    loc += v[k];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __shared__ int64_t ws[kScanThreads / 32];
  if (lane == 31) ws[wid] = incl;
  __syncthreads();
  int64_t wbase = 0;
  for (int w = 0; w < wid; ++w) wbase += ws[w];
  int64_t run = sums[blockIdx.x] + wbase + incl - loc;
#pragma unroll
  for (int k = 0; k < kItemsPerThread; ++k) {
    if (my + k < n) out[my + k] = run;
    run += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanThreads - 1) out[n] = run;
}

// scratch needs compact_blocks(n) int64 entries
inline void scan_counts(const int32_t* in, int64_t n, int64_t* out, int64_t* scratch, cudaStream_t st) {
  int64_t nb = (n + kChunk - 1) / kChunk;
  if (nb == 0) {
    cudaMemsetAsync(out, 0, sizeof(int64_t), st);
    return;
  }
  k_chunk_sums<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, scratch);
  k_scan_i64<<<1, 1024, 0, st>>>(scratch, nb);
  k_chunk_scan<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, scratch, out);
}

}  // namespace ts
