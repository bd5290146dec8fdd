// forward_ws.cuh — K6 forward compositing, warp-specialised (included by composite.cu, which
// provides the record decoding, the error-banded FP32 decisions and the exact FP64 path).
//
// One CTA per 16x16 tile, 288 threads:
//  * warp 8, the PRODUCER, stages the tile list 32 splats at a time into a ring of
//    kWsSlots shared-memory slots: decoded edge functions (stage_q), the splat's rectangle in
//    the tile and its first global pair index (item_off), the colour.  The next chunk's list
//    entries, records and pair bases are loaded while the current one is decoded.
//  * warps 0-7, the CONSUMERS, each own two pixel columns (x = w and w + 8 of the tile, 16
//    rows: interleaved, so every chunk's pairs spread evenly over the consumers).  Per chunk a
//    consumer flattens ITS pixels' (pixel, splat) pairs (rectangle ∩ columns, a warp scan), tests them pair-
//    parallel (A1: face containment, A2: entry / exit and opacity on the compacted
//    candidates), re-decides its own uncertain pairs in exact FP64 (4 lanes per pair), and
//    composites its 32 pixels front to back (lane = pixel) — all warp-synchronous.
//  * slots hand over through mbarriers: full[s] (32 producer arrivals), empty[s] (8 consumer
//    arrivals).  No CTA-wide barrier runs inside the list loop, so a consumer never waits for
//    another block's pairs, staging overlaps compositing, and a block whose 32 pixels all
//    stopped (T < t_stop) leaves the work: it only releases slots until the producer, seeing
//    no active consumer, ends the list.
// Results equal k_forward's (same decisions, same per-pixel blend order and arithmetic): the
// global pair numbering (item_off + rectangle∩tile index) and the pair records the backward
// reads are unchanged.

#ifndef WS_SLOTS
#define WS_SLOTS 4
#endif
#ifndef WS_MINB
#define WS_MINB 3
#endif
#ifndef WS_SLEEP_NS
#define WS_SLEEP_NS 64
#endif

namespace ts {

constexpr int kWsSlots = WS_SLOTS;    // ring depth (chunks of 32 splats)
constexpr int kWsCap = 256;    // pairs per consumer batch (a chunk larger than this is split)
constexpr int kWsConsumers = 8;
constexpr int kWsThreads = 32 * (kWsConsumers + 1);

struct WsSlot {
  Staged st[32];
  float col[32][3];
  int tx0[32], ty0[32], tnx[32];  // splat rectangle ∩ tile: the global pair numbering
  long long ib[32];               // item_off of the splat's list position
  int n;                          // splats in the chunk; -1 = end of the list
  int base;                       // list position of splat 0
};

struct WsWarp {
  float2 code[kWsCap];  // (alpha, 1 - alpha) codes of the batch's blending pairs
  uint16_t exq[kWsCap]; // pairs queued for the exact FP64 re-decision
  uint16_t cq[64];      // A1 candidates (pair | face mask << 8)
  uint8_t jtab[kWsCap]; // splat of each pair of the batch
  uint32_t bmask[32];   // per pixel: splats of the batch that blend (bit j)
  int x0[32], y0[32], nx[32], pre[32];  // splat rectangle ∩ the warp's columns (first column,
                                        // first row, 1 or 2 columns), pair prefix
};

struct WsSmem {
  WsSlot slot[kWsSlots];
  WsWarp w[kWsConsumers];
  unsigned long long full[kWsSlots], empty[kWsSlots];
  int active;  // consumer warps with a pixel still compositing
};

__device__ __forceinline__ uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sh_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sh_addr(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(sh_addr(b)), "r"(parity), "r"(0x989680u)  // suspend up to 10 ms: a waiting warp issues nothing
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  // back off between polls so a waiting warp leaves the issue slots to the working ones
  while (!mbar_try(b, parity)) __nanosleep(WS_SLEEP_NS);
}

template <bool COLOR>
__device__ __forceinline__ void ws_producer(WsSmem& S, const int32_t* __restrict__ list, int L,
                                            const int64_t* __restrict__ ioff, const SplatRec* __restrict__ recs,
                                            const float* __restrict__ colors, int tx0, int ty0) {
  const int lane = threadIdx.x & 31;
  // software pipeline: chunk c's record, list entry and pair base sit in registers while
  // chunk c - 1 is decoded
  int k = lane < L ? __ldg(list + lane) : 0;
  long long ib = lane < L ? __ldg(ioff + lane) : 0;
  float4 q[6];
  if (lane < L) {
    const float4* src = reinterpret_cast<const float4*>(recs + k);
#pragma unroll
    for (int i = 0; i < 6; ++i) q[i] = __ldg(src + i);
  }
  for (int c = 0;; ++c) {
    const int s = c % kWsSlots;
    const int base = c * 32;
    // next chunk's list entry + pair base (independent of this chunk's decode)
    const int nb = base + 32 + lane;
    const int k2 = nb < L ? __ldg(list + nb) : 0;
    const long long ib2 = nb < L ? __ldg(ioff + nb) : 0;
    if (c >= kWsSlots) mbar_wait(&S.empty[s], (unsigned)((c / kWsSlots) - 1) & 1u);
    WsSlot& sl = S.slot[s];
    const bool end = base >= L || *reinterpret_cast<volatile int*>(&S.active) == 0;
    if (end) {
      if (lane == 0) sl.n = -1;
      mbar_arrive(&S.full[s]);
      return;
    }
    const int n = min(32, L - base);
    if (lane < n) {
      Staged& st = sl.st[lane];
      stage_q<true>(q[0], q[1], q[2], q[3], q[4], q[5], k, st);
      int x0, y0, nx, cnt;
      if (!tile_rect(st.rx0, st.rx1, st.ry0, st.ry1, tx0, ty0, x0, y0, nx, cnt)) {
        x0 = y0 = 0;
        nx = 1;
      }
      sl.tx0[lane] = x0;
      sl.ty0[lane] = y0;
      sl.tnx[lane] = nx;
      sl.ib[lane] = ib;
      if (COLOR)
        for (int i = 0; i < 3; ++i) sl.col[lane][i] = __ldg(colors + (int64_t)k * 3 + i);
    }
    if (lane == 0) {
      sl.n = n;
      sl.base = base;
    }
    mbar_arrive(&S.full[s]);
    k = k2;
    ib = ib2;
    if (nb < L) {
      const float4* src = reinterpret_cast<const float4*>(recs + k);
#pragma unroll
      for (int i = 0; i < 6; ++i) q[i] = __ldg(src + i);
    }
  }
}

// one blending pair of a consumer batch: phase-B code, blend bit, global record + bit
__device__ __forceinline__ void ws_put(WsWarp& Wp, const WsSlot& sl, int it, int j, int q, int px, int py,
                                       const Blend& b, uint32_t* __restrict__ pair_bits,
                                       float4* __restrict__ pair_rec) {
  TS_ASSERT(it >= 0 && it < kWsCap && j >= 0 && j < sl.n && q >= 0 && q < 32);
  const float2 c = encode(true, b);
  Wp.code[it] = c;
  atomicOr(&Wp.bmask[q], 1u << j);
  const long long g = sl.ib[j] + (long long)(py - sl.ty0[j]) * sl.tnx[j] + (px - sl.tx0[j]);
  TS_ASSERT(py >= sl.ty0[j] && px >= sl.tx0[j] && px < sl.tx0[j] + sl.tnx[j]);
  pair_rec[g] = make_float4(c.x, c.y, pack_face(b.sp, b.fip), pack_face(b.sn, b.fin));
  atomicOr(pair_bits + (g >> 5), 1u << (g & 31));
}

// pixel of batch pair `it` (batch starts at pair p0 of the chunk): row-major over the splat's
// rows and its (one or two) columns of the warp, 8 pixels apart
__device__ __forceinline__ int ws_pair(const WsWarp& Wp, int it, int p0, int& j, int& px, int& py) {
  j = Wp.jtab[it];
  const int local = it + p0 - Wp.pre[j];
  const int nx = Wp.nx[j];
  const int yy = local >> (nx - 1);
  px = Wp.x0[j] + 8 * (local - yy * nx);
  py = Wp.y0[j] + yy;
  return local;
}
// lane of the warp's pixel (x, y): lane = 2 * row + (column is the second one)
__device__ __forceinline__ int ws_lane(int px, int py, int tx0, int ty0, int w) {
  return 2 * (py - ty0) + ((px - tx0 - w) >> 3);
}

// A2 on up to 32 compacted candidates (one per lane)
__device__ __forceinline__ void ws_a2(WsWarp& Wp, const WsSlot& sl, int m, int p0, int tx0, int ty0, int w, float s,
                                      const Scene64& S64, int& nex, uint32_t* __restrict__ pair_bits,
                                      float4* __restrict__ pair_rec) {
  const int lane = threadIdx.x & 31;
  int e = 0, it = 0;
  if (lane < m) {
    const uint32_t c = Wp.cq[lane];
    it = (int)(c & 255u);
    int j, px, py;
    ws_pair(Wp, it, p0, j, px, py);
    const Staged& r = sl.st[j];
    Blend b;
    e = blend_fast(r, (float)(px - r.rx0) + 0.5f, (float)(py - r.ry0) + 0.5f, s, c >> 8, b);
    if (e == 1) ws_put(Wp, sl, it, j, ws_lane(px, py, tx0, ty0, w), px, py, b, pair_bits, pair_rec);
    if (e == 2) prefetch_exact(S64, r.k);
  }
  const unsigned em = __ballot_sync(0xffffffffu, e == 2);
  if (e == 2) Wp.exq[nex + __popc(em & ((1u << lane) - 1u))] = (uint16_t)it;
  nex += __popc(em);
  __syncwarp();
}

template <bool COLOR>
__global__ void __launch_bounds__(kWsThreads, WS_MINB) k_forward_ws(
    const int32_t* __restrict__ torder, const int64_t* __restrict__ starts, const int32_t* __restrict__ items,
    const int32_t* __restrict__ witems, const uint8_t* __restrict__ nonmono, const SplatRec* __restrict__ recs,
    const float* __restrict__ colors, Scene64 S64, int tiles_x, int W, int H, float s, double s64, float t_stop,
    bool clip_stops, const int64_t* __restrict__ item_off, uint32_t* __restrict__ pair_bits,
    float4* __restrict__ pair_rec, float* __restrict__ normal_map, float* __restrict__ depth_map,
    float* __restrict__ opacity_map, float* __restrict__ color_map, int32_t* __restrict__ n_proc,
    int32_t* __restrict__ n_blend, const int* __restrict__ ovf) {
  if (ovf && *ovf) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WsSmem& S = *reinterpret_cast<WsSmem*>(smem_raw);
  const int tile = torder[blockIdx.x];
  const int tx0 = (tile % tiles_x) * TS_TILE, ty0 = (tile / tiles_x) * TS_TILE;
  const int64_t lo = starts[tile];
  const int L = (int)(starts[tile + 1] - lo);
  const int32_t* list = (nonmono[tile] ? witems : items) + lo;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsSlots; ++i) {
      mbar_init(&S.full[i], 32);
      mbar_init(&S.empty[i], kWsConsumers);
    }
    S.active = kWsConsumers;
  }
  __syncthreads();
  if (warp == kWsConsumers) {
    ws_producer<COLOR>(S, list, L, item_off + lo, recs, colors, tx0, ty0);
    return;
  }
  // ---- consumer: pixel columns warp and warp + 8 of the tile ------------------------------
  WsWarp& Wp = S.w[warp];
  const int cx0 = tx0 + warp;  // first column
  const int xi = cx0 + 8 * (lane & 1), yi = ty0 + (lane >> 1);
  const bool inside = xi < W && yi < H;
  const bool count_pairs = g_ts_debug_flags & 16;
  unsigned npairs = 0;
  float T = 1.f;
  Accum<COLOR> acc;
  acc.zero();
  bool done = !inside;
  int nproc = inside ? L : 0, nb = 0;
  Wp.bmask[lane] = 0u;
  unsigned dmask = __ballot_sync(0xffffffffu, done);
  bool active = dmask != 0xffffffffu;
  if (!active && lane == 0) atomicSub(&S.active, 1);
  for (int c = 0;; ++c) {
    const int sidx = c % kWsSlots;
    mbar_wait(&S.full[sidx], (unsigned)(c / kWsSlots) & 1u);
    const WsSlot& sl = S.slot[sidx];
    const int n = sl.n;
    if (n < 0) break;
    if (active) {
      // this warp's pairs of the chunk: rectangle ∩ the warp's two columns (lane = splat)
      int cnt = 0, x0 = 0, y0 = 0, nx = 1;
      if (lane < n) {
        const Staged& r = sl.st[lane];
        const bool c0 = r.rx0 <= cx0 && cx0 <= r.rx1, c1 = r.rx0 <= cx0 + 8 && cx0 + 8 <= r.rx1;
        y0 = max(r.ry0, ty0);
        const int y1 = min(r.ry1, ty0 + TS_TILE - 1);
        if ((c0 || c1) && y0 <= y1) {
          nx = (int)c0 + (int)c1;
          x0 = c0 ? cx0 : cx0 + 8;
          cnt = nx * (y1 - y0 + 1);
        }
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      Wp.x0[lane] = x0;
      Wp.y0[lane] = y0;
      Wp.nx[lane] = nx;
      Wp.pre[lane] = incl - cnt;
      int j0 = 0;
      while (j0 < n && dmask != 0xffffffffu) {
        const int p0 = __shfl_sync(0xffffffffu, incl - cnt, j0);
        const unsigned okm = __ballot_sync(0xffffffffu, lane >= j0 && lane < n && incl - p0 <= kWsCap);
        const int j1 = 32 - __clz(okm);
        const int P = __shfl_sync(0xffffffffu, incl, j1 - 1) - p0;
        if (lane >= j0 && lane < j1)
          for (int a = incl - cnt - p0, e = incl - p0; a < e; ++a) Wp.jtab[a] = (uint8_t)lane;
        __syncwarp();
        // ---- A: pair-parallel face tests, candidates compacted, A2 32 at a time ----------
        int nex = 0, ncand = 0;
        for (int it0 = 0; it0 < P; it0 += 32) {
          const int it = it0 + lane;
          bool cand = false, ev = false;
          uint32_t fm = 0;
          if (it < P) {
            int j, px, py;
            ws_pair(Wp, it, p0, j, px, py);
            const int q = ws_lane(px, py, tx0, ty0, warp);
            if (!((dmask >> q) & 1u)) {
              ev = true;
              const Staged& r = sl.st[j];
              fm = face_mask(r, (float)(px - r.rx0) + 0.5f, (float)(py - r.ry0) + 0.5f);
              cand = (fm & 16u) || __popc(fm) >= 2;
            }
          }
          if (count_pairs) npairs += __popc(__ballot_sync(0xffffffffu, ev));
          const unsigned cm = __ballot_sync(0xffffffffu, cand);
          if (cand) Wp.cq[ncand + __popc(cm & ((1u << lane) - 1u))] = (uint16_t)(it | (fm << 8));
          ncand += __popc(cm);
          __syncwarp();
          if (ncand >= 32) {
            ws_a2(Wp, sl, 32, p0, tx0, ty0, warp, s, S64, nex, pair_bits, pair_rec);
            const int rest = ncand - 32;
            const uint16_t moved = lane < rest ? Wp.cq[32 + lane] : 0;
            __syncwarp();
            if (lane < rest) Wp.cq[lane] = moved;
            ncand = rest;
            __syncwarp();
          }
        }
        if (ncand > 0) ws_a2(Wp, sl, ncand, p0, tx0, ty0, warp, s, S64, nex, pair_bits, pair_rec);
        // ---- A': exact FP64 re-decisions of this block's uncertain pairs, 8 per pass -----
        for (int q0 = 0; q0 < nex; q0 += 8) {
          const int qi = q0 + (lane >> 2);
          const bool act = qi < nex;
          const int it = act ? Wp.exq[qi] : 0;
          int j, px, py;
          ws_pair(Wp, it, p0, j, px, py);
          Blend b;
          const bool bl = exact_group(S64, act, sl.st[j].k, px, py, s64, b);
          if (act && bl && (lane & 3) == 0)
            ws_put(Wp, sl, it, j, ws_lane(px, py, tx0, ty0, warp), px, py, b, pair_bits, pair_rec);
        }
        __syncwarp();
        // ---- B: lane = pixel, its blending splats in list order ------------------------
        if (!done) {
          unsigned m = Wp.bmask[lane];
          while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1u;
            const int idx = Wp.pre[j] - p0 + (yi - Wp.y0[j]) * Wp.nx[j] + ((xi - Wp.x0[j]) >> 3);
            const float2 cd = Wp.code[idx];
            acc.add(__fmul_rn(T, cd.x), sl.st[j], COLOR ? sl.col[j] : nullptr);
            T = __fmul_rn(T, fabsf(cd.y));
            ++nb;
            // a clipped blend ends the pixel in the FP64 reference whenever
            // 1 - ALPHA_CLIP < t_stop (see k_forward)
            if (T < t_stop || (cd.y < 0.f && clip_stops)) {
              done = true;
              nproc = sl.base + j + 1;
              break;
            }
          }
        }
        Wp.bmask[lane] = 0u;
        dmask = __ballot_sync(0xffffffffu, done);
        j0 = j1;
      }
      if (dmask == 0xffffffffu) {
        active = false;
        if (lane == 0) atomicSub(&S.active, 1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[sidx]);
  }
  if (inside) {
    const int64_t p = (int64_t)yi * W + xi;
    opacity_map[p] = acc.o;
    depth_map[p] = acc.d;
    normal_map[p * 3 + 0] = acc.n[0];
    normal_map[p * 3 + 1] = acc.n[1];
    normal_map[p * 3 + 2] = acc.n[2];
    if (COLOR) {
      color_map[p * 3 + 0] = acc.c[0];
      color_map[p * 3 + 1] = acc.c[1];
      color_map[p * 3 + 2] = acc.c[2];
    }
    n_proc[p] = nproc;
    n_blend[p] = nb;
  }
  if (count_pairs && lane == 0 && npairs) atomicAdd(&g_ts_counters[2], (unsigned long long)npairs);
}

}  // namespace ts
