// composite.cu — K6 forward compositing, K7 backward + vertex chain, N_w window.
//
// One 256-thread CTA per 16x16 tile; the tile's list is processed in chunks of up to kCh
// splats whose (pixel, splat) PAIRS — the pixels of each splat's pixel rectangle inside the
// tile (the reference's inclusive bbox test, _core.pyx:80, made exact at setup) — are
// flattened into one index space of at most kCap pairs.  Every pair of the view has a
// global index: item_off[list position] + local index in the rectangle (k_window_counts).
//
// Forward (forward_tiles, _core.pyx:98-229):
//  A (pair-parallel, dense lanes): hit + opacity of every pair.  FP32 on sign-normalised
//    edge functions in splat-anchored coordinates; any pair within a rigorous FP32 error
//    band of a decision threshold (face edge, alpha = 0, alpha = ALPHA_CLIP, tiny alpha)
//    is re-decided with the reference's exact FP64 arithmetic (below:
//    exact_group / exact_face), so the blended set matches the FP64 reference.  The pair's
//    (alpha, 1-alpha) goes to shared memory for phase B and, with s*sigmoid(-s f) of the
//    entry/exit points and the two face ids, to the global pair records the backward
//    reads — the backward never re-evaluates a hit.
//  B (pixel-serial): each thread blends its pixel's pairs front to back (Eq. 2,
//    _core.pyx:189-213) with early stop at T < t_stop; a finished pixel's later pairs are
//    skipped by phase A; the CTA leaves when all its pixels stopped.
//
// The N_w resorting window (_core.pyx:171-187) pops the same sequence for every pixel of a
// tile — it depends only on the list.  When mean depth is non-decreasing along the list
// (bin.cu flags it) the window is the identity; otherwise k_window replays it per tile.
//
// Backward (backward_tiles _core.pyx:344-471 + splat_grads_to_vertices raster.py:253-306):
//  load: the chunk's pair records (contiguous in global memory) into shared memory;
//  B (pixel-serial, FRONT to back): w = T a and the d_alpha chain
//      G = sum_ch g_ch (T x_ch (1-a) - S_ch),  S_ch = C_final,ch - prefix_ch (inclusive)
//    = the reference's d_alpha * (1 - a) with the suffix sums taken from the forward maps —
//    no division by 1-a, no reverse walk, no per-pixel record lists;
//  C (item-parallel): each warp compacts the blended pairs of its splats (ballot) and
//    processes them 32 at a time — face-hit backward (_core.pyx:295-341) into a 24-float
//    row per item — then a segmented sum into the per-(tile, splat) gradient row, written
//    added (red.global.add.v4.f32) into the splat's row.  k_chain reads each splat's row
//    (coalesced), applies the normal and camera chains and scatters to vertices
//    with one red.global.add.v4.f32 per (splat, vertex).
#include "../../include/tetsplat_b200.h"
#include "internal.cuh"
#include "scan.cuh"

namespace ts {

constexpr float kAlphaClipF = 0.9999f;  // splat.py:14
constexpr float kOneMinusClipF = 1e-4f;
constexpr double kAlphaClipD = 1.0 - 1e-4;  // ALPHA_CLIP in FP64
constexpr int kCh = 64;      // max splats per chunk (one bit each in the per-pixel masks)
constexpr int kCap = 2048;   // max (pixel, splat) pairs per chunk
typedef unsigned long long ChunkMask;

// set bit j of a 64-bit shared mask with a native 32-bit atomic (64-bit shared atomicOr is
// a CAS loop on sm_100)
__device__ __forceinline__ void mask_set(ChunkMask* m, int j) {
  atomicOr(reinterpret_cast<unsigned*>(m) + (j >> 5), 1u << (j & 31));
}
constexpr int kGr = 24;      // floats per (tile, splat) gradient row
constexpr int kWarps = TS_TILE_PX / 32;

struct __align__(16) Staged {
  int rx0, rx1, ry0, ry1;  // pixel rectangle (inclusive, clipped to the image)
  float band;
  uint32_t flags;
  int k;
  float md;
  float iz[4], df[4];  // 1/z; f_i - f_0
  float eux[4], euy[4], cu[4], evx[4], evy[4], cv[4], adet[4];
  float n[3];
  float fband;  // FP32 (f_hit - f0) error <= fband / |det_face| (see stage())
  float ftol0;  // rounding of the stored f deltas
  float f0;
  float pad[2];
};
static_assert(sizeof(Staged) == 208, "Staged must be 208 bytes");

// diagnostics: [0] pairs re-decided in FP64 at a face edge / degenerate face,
// [1] pairs re-decided in FP64 at an alpha threshold, [2] forward pairs evaluated, [3] of [0],
// pairs of splats with a sign-uncertain FP32 face determinant; [4..6] of [1], by reason:
// |f_prev - f_next| within the FP32 f error bound, alpha below the tiny-alpha bound or near
// ALPHA_CLIP; [7] re-decided pairs whose alpha needed the FP64 softplus chain
__device__ unsigned long long g_ts_counters[8];
// diagnostics only (flag bit 64): histograms of how far inside its error bound a re-decided pair
// lies — [0,16): alpha pairs by floor(-log2(|f_prev - f_next| / ftol)), [16,32): edge pairs by
// floor(-log2(|min(u, v, w)| / band)) of the nearest face edge (clamped to 15)
__device__ unsigned long long g_ts_hist[32];
// diagnostics only: bit 0 = skip the exact FP64 re-decisions (timing experiments; breaks parity),
// bit 4 = count the pairs phase A evaluates (g_ts_counters[2]), bit 7 (host side, scene build)
// = no never-blend certificate (the reference's own pair counts for bench.py's work model)
__device__ int g_ts_debug_flags;
static int h_debug_flags = 0;  // host copy of the debug flags
int ts_impl_debug_flags() { return h_debug_flags; }
// diagnostics only (flag bit 1): per-tile forward start/end globaltimer, SM id
__device__ unsigned long long g_ts_tile_time[2 * 65536];
__device__ unsigned int g_ts_tile_sm[65536];

// diagnostics only (flag bit 2): clock64 cycles between the CTA barriers, thread 0 of every
// CTA, summed per phase: [0,4) forward stage/A/A'/B, [8,13) backward stage/load/B/C/write
__device__ unsigned long long g_ts_phase[16];
// (accumulated in shared memory, slot 7 = last stamp, so the hot loop keeps its registers)
#define TS_PHASE(k)                   \
  if (ptime) {                        \
    const long long t_ = clock64();   \
    pacc[k] += t_ - pacc[7];          \
    pacc[7] = t_;                     \
  }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// single-MUFU reciprocal (max 1 ulp error; the FP32 error bands budget for it)
__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// decode one record (prefetched into shared memory) into the chunk's staged form
// FOLD (forward): faces the reference rejects as degenerate get edge functions that are always
// out, so phase A1 needs no validity test
template <bool FOLD>
__device__ __forceinline__ void stage_q(const float4 q0, const float4 q1, const float4 q2, const float4 q3,
                                        const float4 q4, const float4 q5, int k, Staged& s) {
  int rx = __float_as_int(q0.x), ry = __float_as_int(q0.y);
  s.rx0 = (int)(short)(rx & 0xffff);
  s.rx1 = rx >> 16;
  s.ry0 = (int)(short)(ry & 0xffff);
  s.ry1 = ry >> 16;
  s.band = q0.z;
  s.flags = __float_as_uint(q0.w);
  s.k = k;
  const float vx[4] = {q1.x, q1.y, q1.z, q1.w}, vy[4] = {q2.x, q2.y, q2.z, q2.w};
  const float z[4] = {q3.x, q3.y, q3.z, q3.w};
  s.f0 = q4.x;
  s.df[0] = 0.f;
  s.df[1] = q4.y;
  s.df[2] = q4.z;
  s.df[3] = q4.w;
  s.n[0] = q5.x;
  s.n[1] = q5.y;
  s.n[2] = q5.z;
  s.md = q5.w;
#pragma unroll
  for (int v = 0; v < 4; ++v) s.iz[v] = 1.0f / z[v];
#pragma unroll
  for (int fi = 0; fi < 4; ++fi) {
    const int ia = face_vert(fi, 0), ib = face_vert(fi, 1), ic = face_vert(fi, 2);
    float m00 = vx[ib] - vx[ia], m10 = vy[ib] - vy[ia];
    float m01 = vx[ic] - vx[ia], m11 = vy[ic] - vy[ia];
    float det = m00 * m11 - m01 * m10;
    float sd = det < 0.f ? -1.f : 1.f;
    float eux = sd * m11, euy = -sd * m01, evx = -sd * m10, evy = sd * m00;
    s.eux[fi] = eux;
    s.euy[fi] = euy;
    s.evx[fi] = evx;
    s.evy[fi] = evy;
    s.cu[fi] = -(eux * vx[ia] + euy * vy[ia]);
    s.cv[fi] = -(evx * vx[ia] + evy * vy[ia]);
    s.adet[fi] = fabsf(det);
    if (FOLD && !((s.flags >> fi) & 1u)) {  // degenerate in the reference: never contains a pixel
      s.eux[fi] = s.euy[fi] = s.evx[fi] = s.evy[fi] = 0.f;
      s.cu[fi] = s.cv[fi] = -1e30f;
    }
  }
  // f_hit - f0 = sum(lambda_i df_i): with edge-function errors E <= band/16 the barycentric
  // error is <= 4 E (z_max/z_min) / |det|, i.e. 0.25 band zr spread / |det| per face and
  // 0.5 band zr spread / |det| for f_prev - f_next; 0.75 keeps a 1.5x margin.
  float fmax = fmaxf(fabsf(s.df[1]), fmaxf(fabsf(s.df[2]), fabsf(s.df[3])));
  float izmin = fminf(fminf(s.iz[0], s.iz[1]), fminf(s.iz[2], s.iz[3]));
  float izmax = fmaxf(fmaxf(s.iz[0], s.iz[1]), fmaxf(s.iz[2], s.iz[3]));
  s.fband = 0.75f * s.band * (izmax * frcp(izmin)) * fmax;
  s.ftol0 = 1e-6f * fmax;
}

template <bool FOLD>
__device__ __forceinline__ void stage(const SplatRec& rec, int k, Staged& s) {
  const float4* p = reinterpret_cast<const float4*>(&rec);
  stage_q<FOLD>(p[0], p[1], p[2], p[3], p[4], p[5], k, s);
}

struct Hit {
  float fp, fn;  // f - f0 at entry / exit
  int fip, fin;
};

// Phase A1: the faces that certainly contain the pixel (bits 0-3); bit 4 = undecided (within
// the band of a face edge, or a splat with a sign-uncertain face).  The reference's face test:
// a face is out iff min(u, v, w) < -band, in iff min(u, v, w) > band (faces the reference
// rejects as degenerate were given edge functions that are always out, see stage()).
__device__ __forceinline__ uint32_t face_mask(const Staged& s, float px, float py) {
  const float band = s.band;
  uint32_t m = s.flags & 16u;
  float amin = INFINITY;  // smallest |min edge value| over the faces: within the band -> exact path
#pragma unroll
  for (int fi = 0; fi < 4; ++fi) {
    const float u = fmaf(s.eux[fi], px, fmaf(s.euy[fi], py, s.cu[fi]));
    const float v = fmaf(s.evx[fi], px, fmaf(s.evy[fi], py, s.cv[fi]));
    const float w = s.adet[fi] - u - v;
    const float mn = fminf(fminf(u, v), w);
    m |= mn > band ? (1u << fi) : 0u;
    amin = fminf(amin, fabsf(mn));  // (a NaN edge value is ignored by fminf, as by the compares)
  }
  return amin <= band ? (m | 16u) : m;
}

// Phase A2: entry / exit among the in-faces of mask m (face order, first hit seeds, strict
// < / > updates — _splat_hits' rule, _core.pyx:67-95), recomputing each in-face's values.
__device__ __forceinline__ void hit_faces(const Staged& s, float px, float py, uint32_t m, Hit& h) {
  int nh = 0, lo = -1, hi = -1;
  float zlo = 0.f, zhi = 0.f, flo = 0.f, fhi = 0.f;
  for (uint32_t mm = m & 15u; mm; mm &= mm - 1u) {
    const int fi = __ffs(mm) - 1;
    const float u = fmaf(s.eux[fi], px, fmaf(s.euy[fi], py, s.cu[fi]));
    const float v = fmaf(s.evx[fi], px, fmaf(s.evy[fi], py, s.cv[fi]));
    const float w = s.adet[fi] - u - v;
    const int ia = fi == 0 ? 1 : 0, ib = fi <= 1 ? 2 : 1, ic = fi <= 2 ? 3 : 2;
    const float wa = w * s.iz[ia], wb = u * s.iz[ib], wc = v * s.iz[ic];
    const float rD = frcp(wa + wb + wc);
    const float zp = s.adet[fi] * rD;
    const float fh = (wa * s.df[ia] + wb * s.df[ib] + wc * s.df[ic]) * rD;
    if (nh == 0 || zp < zlo) { zlo = zp; flo = fh; lo = fi; }
    if (nh == 0 || zp > zhi) { zhi = zp; fhi = fh; hi = fi; }
    ++nh;
  }
  h.fp = flo;
  h.fn = fhi;
  h.fip = lo;
  h.fin = hi;
}

__device__ __forceinline__ float sigmoidf_stable(float x) {
  if (x >= 0.f) return 1.0f / (1.0f + expf(-x));
  float e = expf(x);
  return e / (1.0f + e);
}

// Outcome of one (pixel, splat) pair.
struct Blend {
  float a, om;    // unclipped alpha and 1 - alpha
  float sp, sn;   // s * sigmoid(-s f_prev), s * sigmoid(-s f_next): d alpha / d f factors
  int fip, fin;   // entry / exit faces
  bool clipped;   // alpha_un > ALPHA_CLIP (no d_alpha/d_f, _core.pyx:462)
};

// One face of the reference's _face_hit (_core.pyx:39-64) in exact FP64 (no contraction); the
// face's vertices a, b, c (projected x, y and depth) are given, F = the splat's SDF samples.
__device__ __forceinline__ bool exact_face(const double* F, int fi, double ax, double ay, double bx, double by,
                                          double cx, double cy, double za, double zb, double zc, double px, double py,
                                          double& zp, double& fh) {
  const int ia = fi == 0 ? 1 : 0, ib = fi <= 1 ? 2 : 1, ic = fi <= 2 ? 3 : 2;
  const double m00 = dsub(bx, ax), m10 = dsub(by, ay);
  const double m01 = dsub(cx, ax), m11 = dsub(cy, ay);
  const double det = dsub(dmul(m00, m11), dmul(m01, m10));
  if (fabs(det) < kEpsDet) return false;
  const double rx = dsub(px, ax), ry = dsub(py, ay);
  const double u = ddiv(dsub(dmul(m11, rx), dmul(m01, ry)), det);
  const double v = ddiv(dadd(dmul(-m10, rx), dmul(m00, ry)), det);
  if (u < 0.0 || v < 0.0 || dadd(u, v) > 1.0) return false;
  const double w0 = ddiv(dsub(dsub(1.0, u), v), za), w1 = ddiv(u, zb), w2 = ddiv(v, zc);
  const double Ss = dadd(dadd(w0, w1), w2);
  fh = ddiv(dadd(dadd(dmul(w0, F[ia]), dmul(w1, F[ib])), dmul(w2, F[ic])), Ss);
  zp = ddiv(1.0, Ss);
  return true;
}

// pull a splat's FP64 scene rows into L1 when one of its pairs is queued for re-decision
__device__ __forceinline__ void prefetch_exact(const Scene64& S, int64_t k) {
  if (S.proj) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.proj + k * 8));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.proj + k * 8 + 7));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.depths + k * 4));
  } else {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.vert_ids + k * 4));
  }
  asm volatile("prefetch.global.L1 [%0];" ::"l"(S.f + k * 4));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(S.bbox + k * 4));
}

// Warp-cooperative exact re-decision (the reference's decision chain, _core.pyx:67-95,
// 35-36, 190-196, in FP64): 4 lanes per queued pair, one face each; the group leader
// combines the faces in face order (first hit seeds, strict < / > updates) and decides
// alpha.  Returns true on the leader when the pair blends.
__device__ __forceinline__ bool exact_group(const Scene64& S, bool act, int64_t k, int xi, int yi, double s, Blend& b) {
  const int lane = threadIdx.x & 31, fi = lane & 3, lead = lane & ~3;
  const double px = xi + 0.5, py = yi + 0.5;
  double zp = 0.0, fh = 0.0;
  bool hit = false;
  const int ia = fi == 0 ? 1 : 0, ib = fi <= 1 ? 2 : 1, ic = fi <= 2 ? 3 : 2;
  double ax, ay, bx, by, cx, cy, za, zb, zc;
  if (S.proj) {
    const double* P = S.proj + k * 8;
    const double* Z = S.depths + k * 4;
    ax = P[2 * ia]; ay = P[2 * ia + 1]; bx = P[2 * ib]; by = P[2 * ib + 1]; cx = P[2 * ic]; cy = P[2 * ic + 1];
    za = Z[ia]; zb = Z[ib]; zc = Z[ic];
  } else {
    // lane fi projects vertex fi of the splat (camera.py:56-67, as the scene build did); the
    // four lanes of the group exchange the three vertices of their faces
    double Pw[3], pc[3], vx, vy, vz;
    vertex_position((uint32_t)S.vert_ids[k * 4 + fi], S.G, S.deform, Pw);
    project_point(S.cam, Pw, vx, vy, vz, pc);
    ax = __shfl_sync(0xffffffffu, vx, lead + ia); ay = __shfl_sync(0xffffffffu, vy, lead + ia);
    bx = __shfl_sync(0xffffffffu, vx, lead + ib); by = __shfl_sync(0xffffffffu, vy, lead + ib);
    cx = __shfl_sync(0xffffffffu, vx, lead + ic); cy = __shfl_sync(0xffffffffu, vy, lead + ic);
    za = __shfl_sync(0xffffffffu, vz, lead + ia); zb = __shfl_sync(0xffffffffu, vz, lead + ib);
    zc = __shfl_sync(0xffffffffu, vz, lead + ic);
  }
  if (act) {
    const double* B = S.bbox + k * 4;
    const bool inb = !(px < B[0] || px > B[2] || py < B[1] || py > B[3]);
    hit = inb && exact_face(S.f + k * 4, fi, ax, ay, bx, by, cx, cy, za, zb, zc, px, py, zp, fh);
  }
  double zlo = 0, zhi = 0, flo = 0, fhi = 0;
  int n = 0, lo = -1, hi = -1;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const bool h = __shfl_sync(0xffffffffu, hit, lead + f);
    const double z = __shfl_sync(0xffffffffu, zp, lead + f);
    const double v = __shfl_sync(0xffffffffu, fh, lead + f);
    if (!h) continue;
    if (n == 0) {
      zlo = zhi = z;
      flo = fhi = v;
      lo = hi = f;
    } else {
      if (z < zlo) { zlo = z; flo = v; lo = f; }
      if (z > zhi) { zhi = z; fhi = v; hi = f; }
    }
    ++n;
  }
  const bool ok = act && n >= 2;
  // The reference blends iff a = 1 - exp(sp(x) - sp(y)) > 0 in FP64, x = -s f_prev,
  // y = -s f_next (these products are bit-identical here).  With alpha = sigmoid(y)(1 - e^{x-y})
  // evaluated in FP32 from the FP64 difference x - y (relative error ~1e-6), the rounded
  // reference outcome is certain once |alpha| clears the rounding of its softplus terms
  // (<= ~4 ulp of max(1, |x|, |y|)) by a wide margin, and alpha is away from ALPHA_CLIP;
  // only the remaining pairs evaluate the FP64 softplus chain (on lanes 1 and 2 at once).
  const double x = dmul(-s, flo), y = dmul(-s, fhi), dxy = dsub(x, y);
  const float yf = (float)y;
  const float ey = expf(-fabsf(yf)), ry = 1.0f / (1.0f + ey);
  const float sy = yf >= 0.f ? ry : ey * ry, sny = yf >= 0.f ? ey * ry : ry;  // sigmoid(+-y)
  const float a_est = sy * -expm1f((float)dxy);
  const float margin = 1e-13f * fmaxf(1.0f, fmaxf(fabsf((float)x), fabsf(yf)));
  const bool certain = fabsf(a_est) > margin && fabsf(a_est - kAlphaClipF) > 1e-5f;
  double spv = 0.0;
  if (ok && !certain && (fi == 1 || fi == 2)) spv = softplus_d(fi == 1 ? x : y);
  const double spx = __shfl_sync(0xffffffffu, spv, lead + 1), spy = __shfl_sync(0xffffffffu, spv, lead + 2);
  if (!ok || fi != 0) return false;
  if ((g_ts_debug_flags & 8) && !certain) atomicAdd(&g_ts_counters[7], 1ull);
  const float sf = (float)s;
  if (certain) {
    if (a_est < 0.f) return false;
    b.a = a_est;
    b.om = fmaf(sy, expf((float)dxy), sny);
    b.clipped = a_est > kAlphaClipF;
  } else {
    const double ed = exp(dsub(spx, spy));
    const double a = dsub(1.0, ed);
    if (a <= 0.0) return false;
    b.a = (float)a;
    b.om = (float)ed;
    b.clipped = a > 1.0 - 1e-4;
  }
  b.sp = sf * sigmoidf_stable(-sf * (float)flo);
  b.sn = sf * sigmoidf_stable(-sf * (float)fhi);
  b.fip = lo;
  b.fin = hi;
  return true;
}

// FP32 fast path with error-bounded decisions: 0 no blend, 1 blend (b filled), 2 the pair
// lies within the error bound of a decision threshold and needs the exact re-decision.
__device__ __forceinline__ int blend_fast(const Staged& r, float px, float py, float s, uint32_t m, Blend& b) {
  Hit h;
  const int e = (m & 16u) ? 2 : (__popc(m) < 2 ? 0 : 1);
  if (e == 0) return 0;
  if (e == 1) hit_faces(r, px, py, m, h);
  if (e == 1) {
    const float dfl = h.fp - h.fn;  // f_prev - f_next, f0 cancels exactly
    const float ftol = r.fband * frcp(fminf(r.adet[h.fip], r.adet[h.fin])) + r.ftol0;
    if (dfl < -ftol) return 0;  // f_prev < f_next: alpha <= 0 exactly
    if (dfl > ftol) {
      // alpha = 1 - exp(sp(x) - sp(y)) = 1 - (1 + e^x) / (1 + e^y), x = -s fp, y = -s fn:
      //   alpha = sigmoid(y) (1 - e^{x-y}),  1 - alpha = sigmoid(-y) + sigmoid(y) e^{x-y}
      // (no logarithms, no cancellation: x - y = -s (fp - fn) from the delta samples)
      const float fn = r.f0 + h.fn;
      const float y = -s * fn, t = s * dfl;
      const float ey = expf(-fabsf(y));
      const float ry = frcp(1.0f + ey);
      const float sy = y >= 0.f ? ry : ey * ry;   // sigmoid(y)
      const float sny = y >= 0.f ? ey * ry : ry;  // sigmoid(-y)
      const float q = expf(-t);                    // e^{x-y}
      const float a_un = sy * (t < 0.25f ? -expm1f(-t) : 1.0f - q);
      // alpha > 1e-10 and not at the clip threshold: the FP64 reference decides the same
      if (a_un > 1e-10f && fabsf(a_un - kAlphaClipF) > 2e-6f) {
        b.a = a_un;
        b.om = fmaf(sy, q, sny);
        b.sn = s * sy;
        // sigmoid(x) = 1 / (1 + e^{-x}), e^{-x} = e^{-y} / q
        b.sp = s * (y >= 0.f ? q * frcp(q + ey) : ey * q * frcp(ey * q + 1.0f));
        b.fip = h.fip;
        b.fin = h.fin;
        b.clipped = a_un > kAlphaClipF;
        return 1;
      }
    }
    atomicAdd(&g_ts_counters[1], 1ull);
    if (g_ts_debug_flags & 64) {
      const float dfl = h.fp - h.fn;
      const float ftol = r.fband * frcp(fminf(r.adet[h.fip], r.adet[h.fin])) + r.ftol0;
      const float q = fabsf(dfl) / ftol;
      const int b = q <= 0.f ? 15 : min(15, max(0, (int)floorf(-log2f(q))));
      atomicAdd(&g_ts_hist[b], 1ull);
    }
    if (g_ts_debug_flags & 8) {
      const float dfl = h.fp - h.fn;
      const float ftol = r.fband * frcp(fminf(r.adet[h.fip], r.adet[h.fin])) + r.ftol0;
      atomicAdd(&g_ts_counters[fabsf(dfl) <= ftol ? 4 : 5], 1ull);
    }
  } else {
    atomicAdd(&g_ts_counters[0], 1ull);
    if (r.flags & 16u) atomicAdd(&g_ts_counters[3], 1ull);
    if (g_ts_debug_flags & 64) {  // the edge value nearest the band among the faces
      float best = 1e30f;
      for (int fi = 0; fi < 4; ++fi) {
        const float u = fmaf(r.eux[fi], px, fmaf(r.euy[fi], py, r.cu[fi]));
        const float v = fmaf(r.evx[fi], px, fmaf(r.evy[fi], py, r.cv[fi]));
        const float w = r.adet[fi] - u - v;
        const float mn = fminf(fminf(u, v), w);
        if (fabsf(mn) <= r.band) best = fminf(best, fabsf(mn));
      }
      const float q = best / r.band;
      const int b = q <= 0.f ? 15 : min(15, max(0, (int)floorf(-log2f(q))));
      atomicAdd(&g_ts_hist[16 + b], 1ull);
    }
  }
  return (g_ts_debug_flags & 1) ? 0 : 2;
}

// Pair code: alpha (+0 bits = no blend, -0 = blended with alpha below FP32 range) and
// 1 - alpha (negative = clipped at ALPHA_CLIP).
__device__ __forceinline__ float2 encode(bool blended, const Blend& b) {
  if (!blended) return make_float2(0.f, 1.f);
  if (b.clipped) return make_float2(kAlphaClipF, -kOneMinusClipF);
  return make_float2(b.a > 0.f ? b.a : -0.f, b.om);
}

// Pair records of the view (item space, written by the forward, read by the backward):
//   pair_bits[g >> 5] bit (g & 31): pair g blends (cleared before the forward);
//   pair_rec[g] = (alpha code, 1 - alpha code, s sigmoid(-s f_prev) | entry face,
//                  s sigmoid(-s f_next) | exit face) for blending pairs only — the face ids
//   ride in the two low mantissa bits (2^-22 relative, far below FP32 gradient noise).
__device__ __forceinline__ float pack_face(float v, int f) {
  return __uint_as_float((__float_as_uint(v) & ~3u) | (unsigned)f);
}
__device__ __forceinline__ int face_of(float v) { return (int)(__float_as_uint(v) & 3u); }
__device__ __forceinline__ bool pair_bit(const uint32_t* __restrict__ bits, int64_t g) {
  return (__ldg(bits + (g >> 5)) >> (g & 31)) & 1u;
}
// OR a warp's 32-pair ballot into the (unaligned) bit range starting at pair g
__device__ __forceinline__ void set_bits(uint32_t* bits, int64_t g, unsigned m) {
  const int sh = (int)(g & 31);
  atomicOr(bits + (g >> 5), m << sh);
  if (sh && (m >> (32 - sh))) atomicOr(bits + (g >> 5) + 1, m >> (32 - sh));
}

template <int NC>
struct Accum {
  float o, d, n[3], c[3];
  __device__ __forceinline__ void zero() {
    o = d = 0.f;
    n[0] = n[1] = n[2] = 0.f;
    c[0] = c[1] = c[2] = 0.f;
  }
  // identical in forward and backward so the backward prefix reproduces C_final exactly
  __device__ __forceinline__ void add(float w, const Staged& r, const float* col) {
    o = __fadd_rn(o, w);
    d = __fmaf_rn(w, r.md, d);
#pragma unroll
    for (int i = 0; i < 3; ++i) n[i] = __fmaf_rn(w, r.n[i], n[i]);
    if (NC)
#pragma unroll
      for (int i = 0; i < 3; ++i) c[i] = __fmaf_rn(w, col[i], c[i]);
  }
};

// rectangle of a splat (packed int16 record rect) inside the tile; false when empty
__device__ __forceinline__ bool tile_rect(int rx0, int rx1, int ry0, int ry1, int tx0, int ty0, int& x0, int& y0,
                                          int& nx, int& cnt) {
  x0 = max(rx0, tx0);
  y0 = max(ry0, ty0);
  const int x1 = min(rx1, tx0 + TS_TILE - 1), y1 = min(ry1, ty0 + TS_TILE - 1);
  if (x0 > x1 || y0 > y1) return false;
  nx = x1 - x0 + 1;
  cnt = nx * (y1 - y0 + 1);
  return true;
}

// Per-chunk pair table.
struct RectTab {
  // per splat, one 16-byte load for the pair decode: .x first pair (exclusive prefix of the
  // pair counts), .y x0 | y0 << 16 (the clipped rectangle's first pixel), .z row length nx,
  // .w 1/nx (float bits)
  int4 rect[kCh];
  int wtot[kCh / 32], wok[kCh / 32];  // staging scan exchange
  int n;             // splats in this chunk
  int total;         // pairs in this chunk
  int64_t ib0;       // global index of the chunk's first pair
  uint8_t jtab[kCap];  // splat of each pair
};

// Next-chunk prefetch (threads [0, kCh)): the list entries of the next chunk are copied
// into shared memory with cp.async at the end of the current chunk's staging, their
// records at the end of the chunk's first phase — both land while the chunk is composited,
// so staging never waits on a dependent global load.  Each thread copies and later consumes
// its own slot.
struct Prefetch {
  SplatRec raw[kCh];
  int32_t idx[kCh];
  int64_t ib0;  // item_off of the next chunk's first list position
#ifdef TS_TMA_RECORDS
  // TMA variant (A/B experiment, profiles/r02_experiments.md): each record is one bulk copy
  // (cp.async.bulk, 96 B) completing on this mbarrier; ph = each staging thread's next parity
  unsigned long long bar;
  uint8_t ph[kCh];
#endif
};
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
#ifdef TS_TMA_RECORDS
__device__ __forceinline__ void tma_wait(Prefetch& P) {
  const unsigned bar = smem_u32(&P.bar), par = P.ph[threadIdx.x];
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(par)
                 : "memory");
  P.ph[threadIdx.x] = (uint8_t)(par ^ 1u);
}
#endif
// threads [0, kCh) before the CTA exits: the one record prefetch still in flight lands first
// (a bulk copy must not write the shared memory of a CTA that has left)
__device__ __forceinline__ void tma_drain(Prefetch& P) {
#ifdef TS_TMA_RECORDS
  if (threadIdx.x < kCh) tma_wait(P);
#else
  (void)P;
#endif
}
// threads [0, kCh), before the first prefetch (TMA variant only)
__device__ __forceinline__ void tma_init(Prefetch& P) {
#ifdef TS_TMA_RECORDS
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  P.ph[threadIdx.x] = 0;
  asm volatile("bar.sync 1, %0;" ::"n"(kCh));
#else
  (void)P;
#endif
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// list entries [pos, pos + min(kCh, avail)) -> P.idx, item_off_tile[pos] -> P.ib0
__device__ __forceinline__ void prefetch_idx(Prefetch& P, const int32_t* __restrict__ list,
                                             const int64_t* __restrict__ item_off_tile, int pos, int avail) {
  const int t = threadIdx.x;
  if (t < min(kCh, avail)) cp_async4(&P.idx[t], list + pos + t);
  if (t == 0 && avail > 0) cp_async8(&P.ib0, item_off_tile + pos);
  cp_async_commit();
}
// records of the prefetched list entries -> P.raw
__device__ __forceinline__ void prefetch_rec(Prefetch& P, const SplatRec* __restrict__ recs, int avail) {
  const int t = threadIdx.x;
  cp_async_wait_all();
#ifdef TS_TMA_RECORDS
  {
    const int m = max(0, min(kCh, avail));
    const unsigned bar = smem_u32(&P.bar);
    if (t == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(m * (int)sizeof(SplatRec))
                   : "memory");
    if (t < m) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // this slot's reads before the async write
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(&P.raw[t])),
          "l"(recs + P.idx[t]), "n"((int)sizeof(SplatRec)), "r"(bar)
          : "memory");
    }
    return;
  }
#endif
  if (t < min(kCh, avail)) {
    const float4* src = reinterpret_cast<const float4*>(recs + P.idx[t]);
    float4* dst = reinterpret_cast<float4*>(&P.raw[t]);
#pragma unroll
    for (int i = 0; i < 6; ++i) cp_async16(dst + i, src + i);
  }
  cp_async_commit();
}

// Threads [0, kCh) only: stage up to kCh prefetched records from list position `base` (at
// most `avail`), cut the chunk so it holds at most kCap pairs, and start the prefetch of the
// next chunk's list entries.  The warps exchange their scan totals through `wtot` behind a
// named barrier over the kCh staging threads.
template <bool FOLD>
__device__ __forceinline__ void stage_chunk(const int32_t* __restrict__ list, int base, int avail, Prefetch& P,
                                            const float* __restrict__ colors, bool color, Staged* sh,
                                            float (*col)[3], RectTab& R, int tx0, int ty0,
                                            const int64_t* __restrict__ item_off_tile) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int m = min(kCh, avail);
  int cnt = 0, x0 = 0, y0 = 0, nx = 1;
  cp_async_wait_all();
#ifdef TS_TMA_RECORDS
  tma_wait(P);
#endif
  if (t < m) {
    const int k = P.idx[t];
    stage<FOLD>(P.raw[t], k, sh[t]);
    const Staged& r = sh[t];
    if (!tile_rect(r.rx0, r.rx1, r.ry0, r.ry1, tx0, ty0, x0, y0, nx, cnt)) {
      nx = 1;
      cnt = 0;
      x0 = y0 = 0;
    }
    if (color)
      for (int c = 0; c < 3; ++c) col[t][c] = colors[(int64_t)k * 3 + c];
  }
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) R.wtot[wid] = v;
  asm volatile("bar.sync 1, %0;" ::"n"(kCh));
  for (int w = 0; w < wid; ++w) v += R.wtot[w];
  if (t < m) R.rect[t] = make_int4(v - cnt, x0 | (y0 << 16), nx, __float_as_int(frcp((float)nx)));
  // cut: the largest prefix with at most kCap pairs (one splat has <= 256 pairs)
  const unsigned ok = __ballot_sync(0xffffffffu, t < m && v <= kCap);
  if (lane == 0) R.wok[wid] = __popc(ok);
  asm volatile("bar.sync 1, %0;" ::"n"(kCh));
  int n = 0;
  for (int w = 0; w < kCh / 32; ++w) n += R.wok[w];
  if (t == n - 1) R.total = v;
  if (t < n) {  // this splat's pair range of the pair -> splat table, word stores in the middle
    int a = v - cnt;
    for (; a < v && (a & 3); ++a) R.jtab[a] = (uint8_t)t;
    const uint32_t pat = (uint32_t)t * 0x01010101u;
    for (; a + 4 <= v; a += 4) *reinterpret_cast<uint32_t*>(&R.jtab[a]) = pat;
    for (; a < v; ++a) R.jtab[a] = (uint8_t)t;
  }
  if (t == 0) {
    R.n = n;
    R.ib0 = P.ib0;
  }
  prefetch_idx(P, list, item_off_tile, base + n, avail - n);
}


__device__ __forceinline__ int pair_splat(const RectTab& R, int it) { return R.jtab[it]; }

// pixel (tile-local index) of pair `it` of splat j
__device__ __forceinline__ void pair_pixel(const RectTab& R, int j, int it, int& xi, int& yi) {
  const int4 r = R.rect[j];
  const int local = it - r.x;
  const int yy = (int)(((float)local + 0.5f) * __int_as_float(r.w));
  xi = (r.y & 0xffff) + (local - yy * r.z);
  yi = (r.y >> 16) + yy;
}

__device__ __forceinline__ int pair_index(const RectTab& R, int j, int xi, int yi) {
  const int4 r = R.rect[j];
  return r.x + (yi - (r.y >> 16)) * r.z + (xi - (r.y & 0xffff));
}

struct FwdSmem {
  Staged sh[kCh];
  float2 code[kCap];  // (alpha, 1 - alpha) per pair of the chunk
  ChunkMask bmask[TS_TILE_PX];  // per pixel: chunk splats that blend (bit j)
  float col[kCh][3];
  uint32_t skip[TS_TILE_PX / 32];
  uint32_t pend[TS_TILE_PX / 32];  // pixels with a pair queued for the exact re-decision
  uint16_t exq[kCap];  // pairs queued for the exact FP64 re-decision
  uint16_t cand[kWarps][64];  // per warp: candidate pairs (it | face mask << 11) of phase A1
  uint32_t cbits[kCap / 32];  // the chunk's blend bits (pair index within the chunk)
  int nex;
  unsigned npairs;  // diagnostics (flag bit 4): pairs evaluated by phase A
  int64_t pair_end;  // checked build: end of the tile's pair range
  RectTab R;
  Prefetch pf;
  long long phase[8];  // diagnostics (flag bit 2)
};

// record one blending pair: shared code + blend bit (forward phase B), the chunk's blend-bit
// word (flushed to pair_bits after the exact re-decisions), global pair record (backward)
__device__ __forceinline__ void put_pair(FwdSmem& F, int it, int j, int q, const Blend& b, int64_t ib0,
                                         float4* __restrict__ pair_rec) {
  TS_ASSERT(it >= 0 && it < F.R.total && j >= 0 && j < F.R.n && q >= 0 && q < TS_TILE_PX);
  TS_ASSERT(ib0 + it < F.pair_end);
  const float2 c = encode(true, b);
  F.code[it] = c;
  mask_set(&F.bmask[q], j);
  atomicOr(&F.cbits[it >> 5], 1u << (it & 31));
  pair_rec[ib0 + it] = make_float4(c.x, c.y, pack_face(b.sp, b.fip), pack_face(b.sn, b.fin));
}

// Phase A2 for one warp: candidates cq[0, m) (pair | face mask << 11), one per lane.
__device__ __forceinline__ void a2_candidates(FwdSmem& F, const uint16_t* cq, int m, const Scene64& S64, float s,
                                              int ty0, int tx0, int64_t ib0, float4* __restrict__ pair_rec) {
  const int lane = threadIdx.x & 31;
  if (lane < m) {
    const uint32_t c = cq[lane];
    const int itc = (int)(c & 2047u);
    const int j = pair_splat(F.R, itc);
    int px_, py_;
    pair_pixel(F.R, j, itc, px_, py_);
    const Staged& r = F.sh[j];
    Blend b;
    const int e = blend_fast(r, (float)(px_ - r.rx0) + 0.5f, (float)(py_ - r.ry0) + 0.5f, s, c >> 11, b);
    if (e == 2) {
      const int slot = atomicAdd(&F.nex, 1);
      TS_ASSERT(slot < kCap);
      F.exq[slot] = (uint16_t)itc;
      const int q = (py_ - ty0) * TS_TILE + (px_ - tx0);
      atomicOr(&F.pend[q >> 5], 1u << (q & 31));
      prefetch_exact(S64, r.k);
    } else if (e == 1) {
      put_pair(F, itc, j, (py_ - ty0) * TS_TILE + (px_ - tx0), b, ib0, pair_rec);
    }
  }
  __syncwarp();
}

template <bool COLOR>
__global__ void __launch_bounds__(TS_TILE_PX, 4) k_forward(
    const int32_t* __restrict__ torder, const int64_t* __restrict__ starts, const int32_t* __restrict__ cpos, const int32_t* __restrict__ witems,
    const int32_t* __restrict__ clen, const SplatRec* __restrict__ recs, const float* __restrict__ colors,
    Scene64 S64, int tiles_x, int W, int H, float s, double s64, float t_stop, bool clip_stops,
    const int64_t* __restrict__ item_off,
    uint32_t* __restrict__ pair_bits, float4* __restrict__ pair_rec, float* __restrict__ normal_map, float* __restrict__ depth_map, float* __restrict__ opacity_map,
    float* __restrict__ color_map, int32_t* __restrict__ n_proc, int32_t* __restrict__ n_blend,
    const int* __restrict__ ovf) {
  if (ovf && *ovf) return;  // the view overflowed its capacities (sync-free path): re-run by the caller
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdSmem& F = *reinterpret_cast<FwdSmem*>(smem_raw);
  if (threadIdx.x == 0) F.npairs = 0;
  const bool count_pairs = g_ts_debug_flags & 16;
  const bool ptime = (g_ts_debug_flags & 4) && threadIdx.x == 0;
  long long* pacc = F.phase;
  if (ptime) {
    for (int k = 0; k < 7; ++k) pacc[k] = 0;
    pacc[7] = clock64();
  }
  const int tile = torder[blockIdx.x];  // longest lists first (k_tile_order)
  const bool timing = (g_ts_debug_flags & 2) && tile < 65536;
  if (timing && threadIdx.x == 0) {
    g_ts_tile_time[2 * tile] = gtimer();
    g_ts_tile_sm[tile] = smid();
  }
  const int tx0 = (tile % tiles_x) * TS_TILE, ty0 = (tile / tiles_x) * TS_TILE;
  const int pix = threadIdx.x;
  const int xi = tx0 + (pix & (TS_TILE - 1)), yi = ty0 + (pix / TS_TILE);
  const bool inside = xi < W && yi < H;
  const int64_t lo = starts[tile];
  // the compositing list: the tile's list (window order) without the splats whose pixel
  // rectangle misses the tile (k_window_counts); cp = their list positions
  const int L = clen[tile];
  const int32_t* list = witems + lo;
  const int32_t* cp = cpos + lo;
#ifdef TS_BOUNDS_CHECKS
  if (threadIdx.x == 0) F.pair_end = item_off[lo + L];
#endif
  float T = 1.f;
  Accum<COLOR> acc;
  acc.zero();
  bool done = !inside;
  int nproc = inside ? (int)(starts[tile + 1] - lo) : 0, nb = 0;
  {
    const unsigned m = __ballot_sync(0xffffffffu, done);
    if ((threadIdx.x & 31) == 0) F.skip[threadIdx.x >> 5] = m;
  }
  if (threadIdx.x < kCh) {
    tma_init(F.pf);
    prefetch_idx(F.pf, list, item_off + lo, 0, L);
    prefetch_rec(F.pf, recs, L);
  }
  for (int base = 0; base < L;) {
    if (threadIdx.x < kCh)
      stage_chunk<true>(list, base, L - base, F.pf, colors, COLOR, F.sh, F.col, F.R, tx0, ty0, item_off + lo);
    F.bmask[pix] = 0ull;
    if (threadIdx.x < kCap / 32) F.cbits[threadIdx.x] = 0u;
    if (threadIdx.x < TS_TILE_PX / 32) F.pend[threadIdx.x] = 0u;
    if (threadIdx.x == 0) F.nex = 0;
    __syncthreads();
    TS_PHASE(0);
    const int n = F.R.n, total = F.R.total;
    const int64_t ib0 = F.R.ib0;
    // ---- A: pair-parallel hit + opacity (FP32, error-bounded) ------------------------------
    //  A1: face containment of every pair (dense lanes); the pairs inside >= 2 faces or within
    //      a band are compacted per warp;  A2: 32 candidates at a time, all lanes busy: entry /
    //      exit interpolation and opacity.  About half of the rectangle pairs miss the splat.
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      uint16_t* cq = F.cand[warp];
      int cnt = 0;
      for (int it0 = warp * 32; it0 < total; it0 += TS_TILE_PX) {
        const int it = it0 + lane;
        bool ev = false, cand = false;
        uint32_t fm = 0;
        if (it < total) {
          const int j = pair_splat(F.R, it);
          int px_, py_;
          pair_pixel(F.R, j, it, px_, py_);
          const int q = (py_ - ty0) * TS_TILE + (px_ - tx0);
          if (!((F.skip[q >> 5] >> (q & 31)) & 1u)) {
            ev = true;
            const Staged& r = F.sh[j];
            fm = face_mask(r, (float)(px_ - r.rx0) + 0.5f, (float)(py_ - r.ry0) + 0.5f);
            cand = (fm & 16u) || __popc(fm) >= 2;
          }
        }
        const unsigned cm = __ballot_sync(0xffffffffu, cand);
        if (count_pairs) {
          const unsigned em = __ballot_sync(0xffffffffu, ev);
          if (lane == 0) atomicAdd(&F.npairs, __popc(em));
        }
        if (cand) cq[cnt + __popc(cm & ((1u << lane) - 1u))] = (uint16_t)(it | (fm << 11));
        cnt += __popc(cm);
        __syncwarp();
        if (cnt >= 32) {
          a2_candidates(F, cq, 32, S64, s, ty0, tx0, ib0, pair_rec);
          const int rest = cnt - 32;
          const uint16_t moved = lane < rest ? cq[32 + lane] : 0;
          __syncwarp();
          if (lane < rest) cq[lane] = moved;
          cnt = rest;
          __syncwarp();
        }
      }
      if (cnt > 0) a2_candidates(F, cq, cnt, S64, s, ty0, tx0, ib0, pair_rec);
    }
    if (threadIdx.x < kCh) prefetch_rec(F.pf, recs, L - base - n);
    __syncthreads();
    TS_PHASE(1);
    // ---- A': exact FP64 re-decisions, 8 pairs per warp, one face per lane ------------------
    //      (F.nex is CTA-uniform after the barrier: chunks without queued pairs skip the pass
    //      and its barrier)
    // ---- B: pixel-serial blend over this pixel's blending splats (bit order = list order) --
    auto blend = [&]() {
      if (done) return;
      ChunkMask m = F.bmask[pix];
      while (m) {
        const int j = __ffsll(m) - 1;
        m &= m - 1ull;
        const float2 c = F.code[pair_index(F.R, j, xi, yi)];
        acc.add(__fmul_rn(T, c.x), F.sh[j], COLOR ? F.col[j] : nullptr);
        T = __fmul_rn(T, fabsf(c.y));
        ++nb;
        // a clipped blend leaves T * (1 - ALPHA_CLIP) < T_STOP in the FP64 reference whenever
        // 1 - ALPHA_CLIP < t_stop (T <= 1), which FP32 T = 1e-4f would not see at T = 1
        if (T < t_stop || (c.y < 0.f && clip_stops)) {
          done = true;
          nproc = cp[base + j] + 1;  // list entries consumed (the reference's position)
          break;
        }
      }
    };
    bool blended = false;
    const int nex = F.nex;
    if (nex > 0) {
      // re-decision batches (8 pairs each) on warps 0, 1, ..; a warp with no batch and no
      // pending pixel blends now, while the re-decisions' FP64 chains run (its codes and masks
      // are final).  (Routing the batches to the warps with pending pixels measured no better.)
      const int warp = threadIdx.x >> 5;
      if (warp * 8 >= nex && F.pend[warp] == 0u) {
        blend();
        blended = true;
      }
      for (int q0 = warp * 8; q0 < nex; q0 += kWarps * 8) {
        const int qi = q0 + ((threadIdx.x & 31) >> 2);
        const bool act = qi < nex;
        const int it = act ? F.exq[qi] : 0;
        const int j = pair_splat(F.R, it);
        int px_, py_;
        pair_pixel(F.R, j, it, px_, py_);
        Blend b;
        const bool bl = exact_group(S64, act, F.sh[j].k, px_, py_, s64, b);
        if (act && bl && (threadIdx.x & 3) == 0)
          put_pair(F, it, j, (py_ - ty0) * TS_TILE + (px_ - tx0), b, ib0, pair_rec);
      }
      __syncthreads();
    }
    TS_PHASE(2);
    // the chunk's blend bits into the view's bit array (words at the chunk ends are shared)
    if (threadIdx.x < (total + 31) / 32) {
      const uint32_t wbits = F.cbits[threadIdx.x];
      if (wbits) set_bits(pair_bits, ib0 + 32 * threadIdx.x, wbits);
    }
    if (ptime) {  // chunks, chunks with re-decisions, re-decided pairs, max per chunk
      pacc[4] += 1;
      pacc[5] += F.nex > 0;
      pacc[6] += F.nex;
      if (F.nex > (int)g_ts_phase[7]) atomicMax(&g_ts_phase[7], (unsigned long long)F.nex);
    }
    if (!blended) blend();
    const unsigned m = __ballot_sync(0xffffffffu, done);
    if ((threadIdx.x & 31) == 0) F.skip[threadIdx.x >> 5] = m;
    base += n;
    const bool all_done = __syncthreads_and(done);
    TS_PHASE(3);
    if (all_done) break;
  }
  tma_drain(F.pf);
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
  if (count_pairs && threadIdx.x == 0) atomicAdd(&g_ts_counters[2], (unsigned long long)F.npairs);
  if (timing && threadIdx.x == 0) g_ts_tile_time[2 * tile + 1] = gtimer();
  if (ptime)
    for (int k = 0; k < 7; ++k) atomicAdd(&g_ts_phase[k], (unsigned long long)pacc[k]);
}


// N_w resorting window (_core.pyx:171-187) for tiles whose list is not mean-depth monotone.
// The list is sorted by (q, splat) with q = 32-bit quantised mean depth, so entries with
// different q are already in strict mean-depth order and every q change is a clean boundary:
// all entries before it are <= all entries after it, so the window pops the whole prefix
// first (ties go to the earlier position) and then restarts with a fresh window.  The
// window therefore acts independently on each run of equal q; runs are short, so one
// thread per run replays the window on it (identity when the run is monotone).
__device__ __forceinline__ uint32_t qkey(double md, double near_, double far_) {
  double qq = ddiv(dsub(md, near_), dsub(far_, near_));
  qq = qq < 0.0 ? 0.0 : qq;
  qq = qq > 1.0 ? 1.0 : qq;
  return (uint32_t)(unsigned long long)dmul(qq, 4294967295.0);  // raster.py:132-134
}

__device__ void window_tile(int t, int64_t lo, int64_t L, const int32_t* __restrict__ items,
                            const double* __restrict__ md, int n_w, double near_, double far_,
                            int32_t* __restrict__ witems, uint32_t* __restrict__ qpos, int32_t* __restrict__ widx_s,
                            double* __restrict__ wz_s, bool q_ready);

// The reference's window (_core.pyx:171-187) replayed over a whole list by one thread (lists
// handed in by a caller that are not sorted by depth key; ts_bins_from_lists flags them 2).
__device__ void window_whole(int64_t lo, int64_t L, const int32_t* __restrict__ items, const double* __restrict__ md,
                             int n_w, int32_t* __restrict__ witems, int32_t* __restrict__ widx_s,
                             double* __restrict__ wz_s) {
  if (threadIdx.x == 0) {
    int32_t* widx = widx_s + lo;
    double* wz = wz_s + lo;
    int64_t wcount = 0, pos = 0, out = 0;
    for (;;) {
      while (wcount < n_w && pos < L) {
        const int32_t k = items[lo + pos++];
        widx[wcount] = k;
        wz[wcount++] = md[k];
      }
      if (wcount == 0) break;
      int64_t m = 0;
      for (int64_t k = 1; k < wcount; ++k)
        if (wz[k] < wz[m]) m = k;
      witems[lo + out++] = widx[m];
      for (int64_t k = m; k < wcount - 1; ++k) {
        widx[k] = widx[k + 1];
        wz[k] = wz[k + 1];
      }
      --wcount;
    }
  }
  __syncthreads();
}

// Window flags of caller-given tile lists: 0 = mean depth non-decreasing (the window is the
// identity), 1 = sorted by the 32-bit depth key but not by mean depth (runs replayed by
// window_tile), 2 = not sorted by depth key (the whole list replayed).  One warp per tile.
__global__ void k_list_flags(int T, const int64_t* __restrict__ starts, const int32_t* __restrict__ items,
                             const double* __restrict__ md, double near_, double far_, uint8_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int64_t lo = starts[t], hi = starts[t + 1];
  bool dec = false, qdec = false;
  for (int64_t i = lo + 1 + lane; i < hi; i += 32) {
    const double a = md[items[i - 1]], b = md[items[i]];
    dec |= b < a;
    qdec |= qkey(b, near_, far_) < qkey(a, near_, far_);
  }
  dec = __any_sync(0xffffffffu, dec);
  qdec = __any_sync(0xffffffffu, qdec);
  if (lane == 0) flags[t] = qdec ? 2 : (dec ? 1 : 0);
}

// SavedState.records of the reference (_core.pyx:206-209, raster.py:94-101) materialised from
// the pair records: per requested tile (CTA) and pixel (thread), the blended splats in blend
// order with their clipped alpha, at rec_off[tile index * 256 + pixel].
__global__ void __launch_bounds__(TS_TILE_PX) k_saved_records(
    const int32_t* __restrict__ tiles, int tiles_x, int W, int H, const int64_t* __restrict__ starts,
    const int32_t* __restrict__ cpos, const int32_t* __restrict__ witems, const int32_t* __restrict__ clen,
    const SplatRec* __restrict__ recs, const int64_t* __restrict__ item_off, const uint32_t* __restrict__ pair_bits,
    const float4* __restrict__ pair_rec, const int32_t* __restrict__ n_proc, const int64_t* __restrict__ rec_off,
    int64_t* __restrict__ idx_out, double* __restrict__ alpha_out) {
  const int tile = tiles[blockIdx.x];
  const int tx0 = (tile % tiles_x) * TS_TILE, ty0 = (tile / tiles_x) * TS_TILE;
  const int xi = tx0 + (threadIdx.x & (TS_TILE - 1)), yi = ty0 + (threadIdx.x / TS_TILE);
  if (xi >= W || yi >= H) return;
  const int64_t lo = starts[tile];
  const int32_t* list = witems + lo;
  const int32_t* cp = cpos + lo;
  const int np = n_proc[(int64_t)yi * W + xi], Lc = clen[tile];
  int64_t o = rec_off[(int64_t)blockIdx.x * TS_TILE_PX + threadIdx.x];
  for (int j = 0; j < Lc && cp[j] < np; ++j) {
    const int k = list[j];
    const int2 rr = *reinterpret_cast<const int2*>(recs + k);
    int x0, y0, nx, c;
    if (!tile_rect((int)(short)(rr.x & 0xffff), rr.x >> 16, (int)(short)(rr.y & 0xffff), rr.y >> 16, tx0, ty0, x0,
                   y0, nx, c))
      continue;
    if (xi < x0 || xi >= x0 + nx || yi < y0 || yi >= y0 + c / nx) continue;
    const int64_t g = item_off[lo + j] + (int64_t)(yi - y0) * nx + (xi - x0);
    TS_ASSERT(g < item_off[lo + j + 1]);
    if (!pair_bit(pair_bits, g)) continue;
    const float4 r = pair_rec[g];
    idx_out[o] = k;
    alpha_out[o] = r.y < 0.f ? kAlphaClipD : (double)fmaxf(r.x, 0.f);
    ++o;
  }
}

// One CTA per tile: the window (non-monotone tiles only), then the pairs per list position
// (|pixel rectangle of the splat ∩ tile|, in the order the compositing kernels walk).
// qpos aliases cnt: each tile's keys are read before its counts overwrite them.
__global__ void __launch_bounds__(256) k_window_counts(int T, int tiles_x, const int64_t* __restrict__ starts,
                                                       const int32_t* __restrict__ items,
                                                       const uint8_t* __restrict__ nonmono,
                                                       const double* __restrict__ md, int n_w, double near_,
                                                       double far_, int32_t* __restrict__ witems,
                                                       const SplatRec* __restrict__ recs, int32_t* __restrict__ cnt,
                                                       int32_t* __restrict__ widx_s, double* __restrict__ wz_s,
                                                       bool q_ready, const int* __restrict__ ovf,
                                                       const int2* __restrict__ prect, int32_t* __restrict__ cpos,
                                                       int32_t* __restrict__ clen) {
  const int t = blockIdx.x;
  if (t >= T || (ovf && *ovf)) return;
  const int64_t lo = starts[t], L = starts[t + 1] - lo;
  const uint8_t flag = nonmono[t];
  const bool nm = flag != 0;
  if (flag == 2)  // a caller-given list not sorted by depth key: the window over the whole list
    window_whole(lo, L, items, md, n_w, witems, widx_s, wz_s);
  else if (nm)
    window_tile(t, lo, L, items, md, n_w, near_, far_, witems, reinterpret_cast<uint32_t*>(cnt), widx_s, wz_s,
                q_ready);
  const int tx0 = (t % tiles_x) * TS_TILE, ty0 = (t / tiles_x) * TS_TILE;
  const int32_t* list = nm ? witems : items;
  // the compositing list: the positions whose pixel rectangle meets the tile (splats certified
  // never to blend have none, records.cuh), in list order, with their list positions (cpos)
  // and pair counts — a stable compaction in rounds of 256 positions, each round reading its
  // entries before any write (witems is compacted in place); the tail counts are zero, so the
  // pair numbering (item_off) is that of the compositing list
  __shared__ int wc[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int kept = 0;
  for (int64_t p0 = 0; p0 < L; p0 += 256) {
    const int64_t p = p0 + threadIdx.x;
    int c = 0, k = 0;
    if (p < L) {
      k = list[lo + p];
      // the 8-byte rectangle: from the compact array when the scene build wrote one (one
      // 32-byte sector holds four), else from the 96-byte record
      const int2 rr = prect ? __ldg(prect + k) : *reinterpret_cast<const int2*>(recs + k);
      int x0, y0, nx;
      tile_rect((int)(short)(rr.x & 0xffff), rr.x >> 16, (int)(short)(rr.y & 0xffff), rr.y >> 16, tx0, ty0, x0, y0,
                nx, c);
    }
    const unsigned m = __ballot_sync(0xffffffffu, c > 0);
    if (lane == 0) wc[warp] = __popc(m);
    __syncthreads();
    int off = kept, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      off += w < warp ? wc[w] : 0;
      tot += wc[w];
    }
    if (c > 0) {
      off += __popc(m & ((1u << lane) - 1u));
      witems[lo + off] = k;
      cpos[lo + off] = (int32_t)p;
      cnt[lo + off] = c;
    }
    kept += tot;
    __syncthreads();
  }
  for (int64_t p = kept + threadIdx.x; p < L; p += blockDim.x) cnt[lo + p] = 0;
  if (threadIdx.x == 0) clen[t] = kept;
}

// the window of one non-monotone tile (all threads of the CTA; ends with a barrier)
__device__ void window_tile(int t, int64_t lo, int64_t L, const int32_t* __restrict__ items,
                            const double* __restrict__ md, int n_w, double near_, double far_,
                            int32_t* __restrict__ witems, uint32_t* __restrict__ qpos, int32_t* __restrict__ widx_s,
                            double* __restrict__ wz_s, bool q_ready) {
  (void)t;
  // the tile's depth keys, once per position (q_ready: the sort already wrote them)
  if (!q_ready) {
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) qpos[lo + i] = qkey(md[items[lo + i]], near_, far_);
    __syncthreads();
  }
  const uint32_t* qs = qpos + lo;
  for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
    const uint32_t qi = qs[i];
    const bool starts_run = i == 0 || qs[i - 1] != qi;
    if (!starts_run) continue;
    if (i + 1 >= L || qs[i + 1] != qi) {  // run of one
      witems[lo + i] = items[lo + i];
      continue;
    }
    int64_t e = i + 1;
    bool mono = true;
    double prev = md[items[lo + i]];
    while (e < L && qs[e] == qi) {
      const double me = md[items[lo + e]];
      mono &= !(me < prev);
      prev = me;
      ++e;
    }
    if (mono) {
      for (int64_t k = i; k < e; ++k) witems[lo + k] = items[lo + k];
      continue;
    }
    int32_t* widx = widx_s + lo + i;
    double* wz = wz_s + lo + i;
    int64_t wcount = 0, pos = i, out = i;
    for (;;) {
      while (wcount < n_w && pos < e) {
        const int32_t k = items[lo + pos];
        widx[wcount] = k;
        wz[wcount] = md[k];
        ++wcount;
        ++pos;
      }
      if (wcount == 0) break;
      int64_t m = 0;
      for (int64_t k = 1; k < wcount; ++k)
        if (wz[k] < wz[m]) m = k;
      witems[lo + out++] = widx[m];
      for (int64_t k = m; k < wcount - 1; ++k) {
        widx[k] = widx[k + 1];
        wz[k] = wz[k + 1];
      }
      --wcount;
    }
  }
  __syncthreads();  // witems complete, the keys (aliasing the counts) consumed
}

// Launch order of the compositing CTAs: tiles by decreasing list length (16-entry buckets),
// so the long tiles start first and the short ones fill the tail (results do not depend on
// the order).  One CTA, shared-memory counting sort.
__global__ void __launch_bounds__(1024) k_tile_order(int T, const int32_t* __restrict__ clen,
                                                    int32_t* __restrict__ order) {
  __shared__ int cnt[1024];
  __shared__ int wsum[32];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  auto bucket = [&](int t) {
    const int L = clen[t];
    return 1023 - (L >> 4 < 1023 ? L >> 4 : 1023);
  };
  for (int t = threadIdx.x; t < T; t += 1024) atomicAdd(&cnt[bucket(t)], 1);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = cnt[threadIdx.x];
  int v = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  int off = 0;
  for (int k = 0; k < w; ++k) off += wsum[k];
  __syncthreads();
  cnt[threadIdx.x] = off + v - c;  // exclusive offset of the bucket
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += 1024) order[atomicAdd(&cnt[bucket(t)], 1)] = t;
}


// backward of one face hit (_core.pyx:295-341) accumulated into an item row (shared memory,
// per-vertex slots: [0,4) d_f, [4,8) d_depth, [8,12) d_px, [12,16) d_py)
__device__ __forceinline__ void face_bwd(float (&acc)[16], const Staged& r, int fi, float px, float py, float g) {
  const int ia = fi == 0 ? 1 : 0, ib = fi <= 1 ? 2 : 1, ic = fi <= 2 ? 3 : 2;
  const float inv_ad = frcp(r.adet[fi]);
  const float eux = r.eux[fi], euy = r.euy[fi], evx = r.evx[fi], evy = r.evy[fi];
  const float u = fmaf(eux, px, fmaf(euy, py, r.cu[fi])) * inv_ad;
  const float v = fmaf(evx, px, fmaf(evy, py, r.cv[fi])) * inv_ad;
  const float wbar = 1.0f - u - v;
  const float iza = r.iz[ia], izb = r.iz[ib], izc = r.iz[ic];
  const float fa = r.df[ia], fb = r.df[ib], fc = r.df[ic];
  const float w0 = wbar * iza, w1 = u * izb, w2 = v * izc;
  const float iS = frcp(w0 + w1 + w2);
  const float fh = (w0 * fa + w1 * fb + w2 * fc) * iS;
  const float dw0 = g * (fa - fh) * iS, dw1 = g * (fb - fh) * iS, dw2 = g * (fc - fh) * iS;
  const float gu = -dw0 * iza + dw1 * izb;
  const float gv = -dw0 * iza + dw2 * izc;
  const float qx = (eux * gu + evx * gv) * inv_ad;
  const float qy = (euy * gu + evy * gv) * inv_ad;
  // per face vertex (a, b, c): d f, d depth, d px, d py
  const float c[4][3] = {{g * w0 * iS, g * w1 * iS, g * w2 * iS},
                         {dw0 * (-w0 * iza), dw1 * (-w1 * izb), dw2 * (-w2 * izc)},
                         {-qx * wbar, -qx * u, -qx * v},
                         {-qy * wbar, -qy * u, -qy * v}};
  // scatter to the tet's vertex slots (face fi omits vertex fi) with selects, so the
  // accumulators stay in registers
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    acc[4 * q + 0] += fi == 0 ? 0.f : c[q][0];
    acc[4 * q + 1] += fi == 0 ? c[q][0] : (fi == 1 ? 0.f : c[q][1]);
    acc[4 * q + 2] += fi <= 1 ? c[q][1] : (fi == 2 ? 0.f : c[q][2]);
    acc[4 * q + 3] += fi == 3 ? 0.f : c[q][2];
  }
}

template <bool COLOR>
struct BwdSmem {
  static constexpr int NC = COLOR ? 23 : 20;  // gradient components per item / (tile, splat) row
  static constexpr int RS = COLOR ? 25 : 21;  // odd item-row stride: conflict-free per-lane rows
  static constexpr int AS = COLOR ? 24 : 20;  // accumulator row stride (whole float4s)
  static constexpr int GM = COLOR ? 7 : 4;    // map gradients per pixel (normal, depth, colour)
  Staged sh[kCh];
  float2 wg[kCap];      // items only — load: (alpha, 1-alpha); phase B: (w = T a, G)
  float col[COLOR ? kCh : 1][3];  // colour variant only
  union {
    ChunkMask bmask[TS_TILE_PX];  // load + B: per pixel, chunk splats that blend (bit j)
    float rows[kWarps][32][RS];   // C: per-item rows of each warp's batch
  } u;
  uint16_t items[kCap];  // C: the chunk's items (pair index) in pair order
  int wcnt[kCap / 32];   // items per 32-pair block -> exclusive offsets
  uint32_t lbits[kCap / 32];  // loaded (blending, not early-stopped) pairs, block k*8+warp
  uint32_t wpre[kCap / 32 + 1];  // the chunk's blend-bit words, loaded by warps 2-4 during staging
  int lim[TS_TILE_PX];   // per pixel: list entries the forward consumed (n_proc)
  float gmap[TS_TILE_PX][GM];  // per pixel: dL/d(normal xyz, depth, colour) — read by phase C
  RectTab R;
  Prefetch pf;
  long long phase[8];  // diagnostics (flag bit 2)
  int maxproc, nitems;
  int64_t pair_end;  // checked build: end of the tile's pair range
};

// occupancy the launch bounds assume (228 KB shared memory per SM, 1 KB reserved per CTA)
static_assert(4 * (sizeof(FwdSmem) + 1024) <= 228 * 1024, "forward: 4 CTAs per SM");
static_assert(3 * (sizeof(BwdSmem<false>) + 1024) <= 228 * 1024, "backward: 3 CTAs per SM");




// One warp, items [b0, b0 + m) of the chunk: face-hit backward of every item into its row,
// then per run of equal splat (items are in pair order, i.e. grouped by splat) one lane per
// component sums the run and adds it to the splat's global row (zeroed per view) with one
// RED.ADD.F32 — a splat's runs (in other batches, chunks and tiles) meet in L2; FP32 order
// noise only, or int64 fixed point when DET (order-independent).
template <bool COLOR, bool DET>
__device__ __forceinline__ void process_batch(BwdSmem<COLOR>& S, int b0, int m, const float4* __restrict__ pair_rec,
                                              int64_t ib0, float* __restrict__ rows,
                                              unsigned long long* __restrict__ fx_bad) {
  using SM = BwdSmem<COLOR>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* row = S.u.rows[warp][lane];
  const int it = lane < m ? (int)S.items[b0 + lane] : 0;
  const int jl = lane < m ? (int)S.R.jtab[it] : -1;
  if (lane < m) {
    const int j = jl;
    const Staged& r = S.sh[j];
    int xi, yi;
    pair_pixel(S.R, j, it, xi, yi);
    const float2 wg = S.wg[it];
    const float w = wg.x, G = wg.y;
    const float* gm = S.gmap[(yi & (TS_TILE - 1)) * TS_TILE + (xi & (TS_TILE - 1))];
#pragma unroll
    for (int i = 0; i < SM::GM; ++i) row[16 + i] = gm[i] * w;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    if (G != 0.f) {
      const float2 sg = __ldg(reinterpret_cast<const float2*>(pair_rec + ib0 + it) + 1);
      const float px = (float)(xi - r.rx0) + 0.5f, py = (float)(yi - r.ry0) + 0.5f;
      face_bwd(acc, r, face_of(sg.x), px, py, G * sg.x);
      face_bwd(acc, r, face_of(sg.y), px, py, -G * sg.y);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) row[i] = acc[i];
  }
  const int jprev = __shfl_up_sync(0xffffffffu, jl, 1);
  unsigned heads = __ballot_sync(0xffffffffu, lane < m && (lane == 0 || jl != jprev));
  __syncwarp();
  while (heads) {
    const int s0 = __ffs(heads) - 1;
    heads &= heads - 1u;
    const int e0 = heads ? __ffs(heads) - 1 : m;
    const int jj = __shfl_sync(0xffffffffu, jl, s0);
    if (lane < SM::NC) {
      float sum = 0.f;
      for (int i = s0; i < e0; ++i) sum += S.u.rows[warp][i][lane];
      if (DET)  // fixed point straight into the splat's row: order-independent
        fx_add(reinterpret_cast<long long*>(rows) + (int64_t)S.sh[jj].k * SM::AS + lane, sum, fx_bad);
      else if (sum != 0.f)  // RED.ADD.F32 straight into the splat's row (L2)
        atomicAdd(rows + (int64_t)S.sh[jj].k * SM::AS + lane, sum);
    }
  }
  __syncwarp();
}

template <bool COLOR, bool DET>
__global__ void __launch_bounds__(TS_TILE_PX, 3) k_backward(
    const int32_t* __restrict__ torder, const int64_t* __restrict__ starts, const int32_t* __restrict__ cpos, const int32_t* __restrict__ witems,
    const int32_t* __restrict__ clen, const SplatRec* __restrict__ recs, const float* __restrict__ colors,
    int tiles_x, int W, int H, const int64_t* __restrict__ item_off, const uint32_t* __restrict__ pair_bits,
    const float4* __restrict__ pair_rec, const float* __restrict__ normal_map,
    const float* __restrict__ depth_map, const float* __restrict__ opacity_map, const float* __restrict__ color_map,
    const float* __restrict__ d_normal, const float* __restrict__ d_depth, const float* __restrict__ d_opacity,
    const float* __restrict__ d_color, const int32_t* __restrict__ n_proc, float* __restrict__ rows,
    float* __restrict__ status, const int* __restrict__ ovf, unsigned long long* __restrict__ fx_bad) {
  if (ovf && *ovf) {  // an overflowed sync-free view: flagged for the step's Adam guard
    if (status && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(status + 2, 1.0f);
    return;
  }
  using SM = BwdSmem<COLOR>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& S = *reinterpret_cast<SM*>(smem_raw);
  const bool ptime = (g_ts_debug_flags & 4) && threadIdx.x == 0;
  long long* pacc = S.phase;
  if (ptime)
    for (int k = 0; k < 7; ++k) pacc[k] = 0;
  const int tile = torder[blockIdx.x];  // longest lists first (k_tile_order)
  const int tx0 = (tile % tiles_x) * TS_TILE, ty0 = (tile / tiles_x) * TS_TILE;
  const int pix = threadIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int xi = tx0 + (pix & (TS_TILE - 1)), yi = ty0 + (pix / TS_TILE);
  const bool inside = xi < W && yi < H;
  const int64_t lo = starts[tile];
  const int32_t* list = witems + lo;  // the compositing list (k_window_counts)
  const int64_t p = inside ? (int64_t)yi * W + xi : 0;
  const int np_list = inside ? n_proc[p] : 0;
#ifdef TS_BOUNDS_CHECKS
  if (threadIdx.x == 0) S.pair_end = item_off[starts[tile + 1]];
  TS_ASSERT(np_list >= 0 && np_list <= starts[tile + 1] - lo);
#endif
  // list entries consumed -> compositing-list entries consumed: entries with list position
  // below n_proc (cpos increases along the compositing list)
  int nproc = 0;
  if (np_list > 0) {
    const int32_t* cp = cpos + lo;
    int a = 0, b = clen[tile];
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (__ldg(cp + mid) < np_list) a = mid + 1;
      else b = mid;
    }
    nproc = a;
  }
  if (threadIdx.x == 0) S.maxproc = 0;
  S.lim[pix] = nproc;
  __syncthreads();
  if (nproc > 0) atomicMax(&S.maxproc, nproc);
  float g_o = 0.f, g_d = 0.f, g_n[3] = {0.f, 0.f, 0.f}, g_c[3] = {0.f, 0.f, 0.f};
  float C_o = 0.f, C_d = 0.f, C_n[3] = {0.f, 0.f, 0.f}, C_c[3] = {0.f, 0.f, 0.f};
  if (inside) {
    g_o = d_opacity[p];
    g_d = d_depth[p];
    C_o = opacity_map[p];
    C_d = depth_map[p];
    for (int i = 0; i < 3; ++i) {
      g_n[i] = d_normal[p * 3 + i];
      C_n[i] = normal_map[p * 3 + i];
      if (COLOR) {
        g_c[i] = d_color[p * 3 + i];
        C_c[i] = color_map[p * 3 + i];
      }
    }
  }
  S.gmap[pix][0] = g_n[0];
  S.gmap[pix][1] = g_n[1];
  S.gmap[pix][2] = g_n[2];
  S.gmap[pix][3] = g_d;
  if (COLOR) {
    S.gmap[pix][4] = g_c[0];
    S.gmap[pix][5] = g_c[1];
    S.gmap[pix][6] = g_c[2];
  }
  if (status) {  // raster.py:209-211: non-finite incoming map gradients, raised by the caller
    bool bad = !isfinite(g_o) || !isfinite(g_d) || !isfinite(g_n[0]) || !isfinite(g_n[1]) || !isfinite(g_n[2]);
    if (COLOR) bad |= !isfinite(g_c[0]) || !isfinite(g_c[1]) || !isfinite(g_c[2]);
    if (__ballot_sync(0xffffffffu, bad) && lane == 0) atomicAdd(status, 1.0f);
  }
  __syncthreads();
  const int maxproc = S.maxproc;
  float T = 1.f;
  Accum<COLOR> P;
  P.zero();
  if (ptime) pacc[7] = clock64();
  if (threadIdx.x < kCh) {
    tma_init(S.pf);
    prefetch_idx(S.pf, list, item_off + lo, 0, maxproc);
    prefetch_rec(S.pf, recs, maxproc);
  }
  // last blend-bit word of the tile's pair range (bounds the word prefetch)
  const int64_t wlast = maxproc > 0 ? (item_off[starts[tile + 1]] - 1) >> 5 : 0;
  for (int base = 0; base < maxproc;) {
    if (threadIdx.x < kCh) {
      stage_chunk<false>(list, base, maxproc - base, S.pf, colors, COLOR, S.sh, S.col, S.R, tx0, ty0, item_off + lo);
    } else if (threadIdx.x < kCh + kCap / 32 + 1) {
      // the chunk's blend-bit words (at most kCap pairs from its first pair), loaded while the
      // staging warps decode: the load phase reads them from shared memory
      const int64_t w = (__ldg(item_off + lo + base) >> 5) + (threadIdx.x - kCh);
      S.wpre[threadIdx.x - kCh] = w <= wlast ? __ldg(pair_bits + w) : 0u;
    }
    S.u.bmask[pix] = 0ull;
    __syncthreads();
    TS_PHASE(0);
    const int n = S.R.n, total = S.R.total;
    const int nblk = (total + TS_TILE_PX - 1) / TS_TILE_PX;  // <= kCap / 256
    const int64_t ib0 = S.R.ib0;
    // ---- load: blend bits (all words first), then the blending, not early-stopped pairs'
    //      codes by cp.async; per-pixel masks; per-32-pair item counts -------------------------
    {
      uint32_t wv[kCap / TS_TILE_PX];
#pragma unroll
      for (int k = 0; k < kCap / TS_TILE_PX; ++k) {
        const int it = threadIdx.x + k * TS_TILE_PX;
        wv[k] = (k < nblk && it < total) ? S.wpre[((ib0 + it) >> 5) - (ib0 >> 5)] : 0u;
      }
#pragma unroll
      for (int k = 0; k < kCap / TS_TILE_PX; ++k) {
        if (k < nblk) {
          const int it = threadIdx.x + k * TS_TILE_PX;
          bool bl = false;
          if (it < total && ((wv[k] >> ((ib0 + it) & 31)) & 1u)) {
            const int j = pair_splat(S.R, it);
            int px_, py_;
            pair_pixel(S.R, j, it, px_, py_);
            const int q = (py_ - ty0) * TS_TILE + (px_ - tx0);
            if (base + j < S.lim[q]) {  // past the pixel's early stop: not composited
              TS_ASSERT(ib0 + it < S.pair_end && it < kCap && j < S.R.n);
              cp_async8(&S.wg[it], pair_rec + ib0 + it);
              mask_set(&S.u.bmask[q], j);
              bl = true;
            }
          }
          const unsigned bm = __ballot_sync(0xffffffffu, bl);
          if (lane == 0) {
            S.wcnt[k * kWarps + warp] = __popc(bm);
            S.lbits[k * kWarps + warp] = bm;
          }
        }
      }
    }
    cp_async_wait_all();
    if (threadIdx.x < kCh) prefetch_rec(S.pf, recs, maxproc - base - n);
    __syncthreads();
    TS_PHASE(1);
    // ---- B: pixel-serial prefix walk over this pixel's blended splats -> (w, G) --------------
    //      (warp 0 first turns the item counts into offsets)
    if (warp == 0) {
      const int nb = nblk * kWarps;  // <= 64 blocks, two per lane
      const int c0 = 2 * lane < nb ? S.wcnt[2 * lane] : 0, c1 = 2 * lane + 1 < nb ? S.wcnt[2 * lane + 1] : 0;
      int v = c0 + c1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (2 * lane < nb) S.wcnt[2 * lane] = v - c0 - c1;
      if (2 * lane + 1 < nb) S.wcnt[2 * lane + 1] = v - c1;
      if (lane == 31) S.nitems = v;
    }
    for (ChunkMask m = S.u.bmask[pix]; m;) {
      const int j = __ffsll(m) - 1;
      m &= m - 1ull;
      const int it = pair_index(S.R, j, xi, yi);
      const float2 c = S.wg[it];
      const float a = c.x, om = fabsf(c.y);
      const bool cl = c.y < 0.f;
      const Staged& r = S.sh[j];
      const float* col = COLOR ? S.col[j] : nullptr;
      const float w = __fmul_rn(T, a);
      P.add(w, r, col);
      float G = 0.f;
      if (!cl) {
        const float Tom = T * om;
        G = g_o * (Tom - (C_o - P.o)) + g_d * (Tom * r.md - (C_d - P.d));
#pragma unroll
        for (int i = 0; i < 3; ++i) G += g_n[i] * (Tom * r.n[i] - (C_n[i] - P.n[i]));
        if (COLOR)
#pragma unroll
          for (int i = 0; i < 3; ++i) G += g_c[i] * (Tom * col[i] - (C_c[i] - P.c[i]));
      }
      S.wg[it] = make_float2(w == 0.f ? -0.f : w, G);
      T = __fmul_rn(T, om);
    }
    __syncthreads();
    TS_PHASE(2);
    // ---- C: the chunk's items in pair order, 32 per warp-batch, batches round-robin ---------
#pragma unroll
    for (int k = 0; k < kCap / TS_TILE_PX; ++k) {
      if (k < nblk) {
        const int it = threadIdx.x + k * TS_TILE_PX;
        const unsigned bm = S.lbits[k * kWarps + warp];
        const bool has = (bm >> lane) & 1u;
        if (has) S.items[S.wcnt[k * kWarps + warp] + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)it;
      }
    }
    __syncthreads();
    const int nitems = S.nitems;
    for (int b0 = warp * 32; b0 < nitems; b0 += TS_TILE_PX)
      process_batch<COLOR, DET>(S, b0, min(32, nitems - b0), pair_rec, ib0, rows, fx_bad);
    __syncthreads();
    TS_PHASE(3);
    base += n;
    TS_PHASE(4);
  }
  tma_drain(S.pf);
  if (ptime)
    for (int k = 0; k < 5; ++k) atomicAdd(&g_ts_phase[8 + k], (unsigned long long)pacc[k]);
}

// per-splat gather + normal chain + camera chain (raster.py:253-306).  FP32 chain math (the
// gradients are FP32); vertex positions are formed in FP64 (grid coordinate + deformation)
// and only their differences / camera-space coordinates are rounded, one vertex at a time.
template <bool COLOR, bool DET>
__global__ void __launch_bounds__(128, 6) k_chain(int64_t K, const float* __restrict__ rows,
                                               const int32_t* __restrict__ vert_ids,
                                               const int32_t* __restrict__ tet_ids, const double* __restrict__ fsc,
                                               const double* __restrict__ deform, Grid G, Camera cam,
                                               float* __restrict__ d_vert, float* __restrict__ d_color,
                                               const int64_t* __restrict__ Kdev, const int* __restrict__ ovf,
                                               Fx fxo, const SplatRec* __restrict__ recs) {
  if (ovf && *ovf) return;
  if (Kdev) K = min(K, *Kdev);
  constexpr int NQ = COLOR ? 6 : 5;  // float4s of a row that carry data
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    // a splat with an empty pixel rectangle (certified never to blend, records.cuh) was never
    // composited: its row is zero
    if (rect_empty(__ldg(reinterpret_cast<const int2*>(recs + k)))) continue;
    float a[4 * NQ];
    if (DET) {  // fixed-point rows (k_backward<DET>)
      const longlong2* src = reinterpret_cast<const longlong2*>(rows) + k * (2 * NQ);
#pragma unroll
      for (int i = 0; i < 2 * NQ; ++i) {
        const longlong2 q = src[i];
        a[2 * i] = fx_value(q.x);
        a[2 * i + 1] = fx_value(q.y);
      }
    } else {
      const float4* src = reinterpret_cast<const float4*>(rows + k * (4 * NQ));
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const float4 q = __ldg(src + i);
        a[4 * i] = q.x;
        a[4 * i + 1] = q.y;
        a[4 * i + 2] = q.z;
        a[4 * i + 3] = q.w;
      }
    }
    const int4 vv = __ldg(reinterpret_cast<const int4*>(vert_ids) + k);
    const uint32_t vid[4] = {(uint32_t)vv.x, (uint32_t)vv.y, (uint32_t)vv.z, (uint32_t)vv.w};
    TS_ASSERT(vid[0] < (uint32_t)(G.n * G.n * G.n) && vid[1] < (uint32_t)(G.n * G.n * G.n) &&
              vid[2] < (uint32_t)(G.n * G.n * G.n) && vid[3] < (uint32_t)(G.n * G.n * G.n));
    const double2 fa = __ldg(reinterpret_cast<const double2*>(fsc) + 2 * k);
    const double2 fb = __ldg(reinterpret_cast<const double2*>(fsc) + 2 * k + 1);
    float e[3][3], pcs[4][3];
    {
      double P0[3];
      vertex_position(vid[0], G, deform, P0);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        double P[3];
        if (v == 0) {
          P[0] = P0[0]; P[1] = P0[1]; P[2] = P0[2];
        } else {
          vertex_position(vid[v], G, deform, P);
          for (int i = 0; i < 3; ++i) e[v - 1][i] = (float)(P[i] - P0[i]);
        }
        for (int r = 0; r < 3; ++r)
          pcs[v][r] = (float)(P[0] * cam.R[r * 3] + P[1] * cam.R[r * 3 + 1] + P[2] * cam.R[r * 3 + 2] + cam.t[r]);
      }
    }
    float dF[4], dPos[4][3];
    const float dMd = a[19];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      dF[v] = a[v];
      dPos[v][0] = dPos[v][1] = dPos[v][2] = 0.f;
    }
    // normal chain: n = g/|g|, dL/dg = (I - n n^T) dL/dn / |g|, dL/df = B^-T [dL/dg, 0]
    // (B^-T [dL/dg, 0] in the cross-product form of _core.pyx:517-541)
    const float df1 = (float)(fa.y - fa.x), df2 = (float)(fb.x - fa.x), df3 = (float)(fb.y - fa.x);
    const float* e1 = e[0];
    const float* e2 = e[1];
    const float* e3 = e[2];
    const float c1[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2], e2[0] * e3[1] - e2[1] * e3[0]};
    const float c2[3] = {e3[1] * e1[2] - e3[2] * e1[1], e3[2] * e1[0] - e3[0] * e1[2], e3[0] * e1[1] - e3[1] * e1[0]};
    const float c3[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const float det = e1[0] * c1[0] + e1[1] * c1[1] + e1[2] * c1[2];
    if (det != 0.f) {
      const float idet = 1.0f / det;
      float g[3];
      for (int i = 0; i < 3; ++i) g[i] = (df1 * c1[i] + df2 * c2[i] + df3 * c3[i]) * idet;
      const float gn = sqrtf(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
      if (gn >= 1e-8f) {
        const float ign = 1.0f / gn;
        const float nn[3] = {g[0] * ign, g[1] * ign, g[2] * ign};
        const float dn[3] = {a[16], a[17], a[18]};
        const float dot = nn[0] * dn[0] + nn[1] * dn[1] + nn[2] * dn[2];
        float dg[3];
        for (int i = 0; i < 3; ++i) dg[i] = (dn[i] - nn[i] * dot) * ign;
        const float d1 = (c1[0] * dg[0] + c1[1] * dg[1] + c1[2] * dg[2]) * idet;
        const float d2 = (c2[0] * dg[0] + c2[1] * dg[1] + c2[2] * dg[2]) * idet;
        const float d3 = (c3[0] * dg[0] + c3[1] * dg[1] + c3[2] * dg[2]) * idet;
        const float dfn[4] = {-(d1 + d2 + d3), d1, d2, d3};
        for (int v = 0; v < 4; ++v) {
          dF[v] += dfn[v];
          for (int i = 0; i < 3; ++i) dPos[v][i] -= dfn[v] * g[i];
        }
      }
    }
    // camera chain: pixel = (fx X/Z + cx, fy Y/Z + cy), depth = Z
    const float fx = (float)cam.fx, fy = (float)cam.fy;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float* pc = pcs[v];
      const float dPx = a[8 + v], dPy = a[12 + v], dZ = a[4 + v] + 0.25f * dMd;
      const float iZ = 1.0f / pc[2];
      const float dpc[3] = {dPx * fx * iZ, dPy * fy * iZ, (-dPx * fx * pc[0] - dPy * fy * pc[1]) * iZ * iZ + dZ};
      for (int j = 0; j < 3; ++j)
        dPos[v][j] += dpc[0] * (float)cam.R[j] + dpc[1] * (float)cam.R[3 + j] + dpc[2] * (float)cam.R[6 + j];
      if (DET)
        fx_add4(fxo.vert + (size_t)vid[v] * 4, dF[v], dPos[v][0], dPos[v][1], dPos[v][2], fxo.bad);
      else
        red_add_v4(d_vert + (size_t)vid[v] * 4, dF[v], dPos[v][0], dPos[v][1], dPos[v][2]);
    }
    if (COLOR) {
      const int64_t t = tet_ids[k];
      for (int c = 0; c < 3; ++c) {
        if (DET)
          fx_add(fxo.color + t * 3 + c, a[20 + c], fxo.bad);
        else
          atomicAdd(d_color + t * 3 + c, a[20 + c]);
      }
    }
  }
}

}  // namespace ts

using namespace ts;

// window-resorted lists + pair offsets of the view: item_off[M+1]; returns the pair count
// a caller-owned temporary when given, else one from the stream-ordered pool (freed by put_tmp)
template <class T>
static T* take_tmp(T* given, size_t n, cudaStream_t st) {
  if (given) return given;
  T* p = nullptr;
  cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), st);
  return p;
}
template <class T>
static void put_tmp(T* p, const T* given, cudaStream_t st) {
  if (p && p != given) cudaFreeAsync(p, st);
}

// q_ready: scr->cnt already holds each position's depth key (written by the sort)
int64_t ts_impl_forward_prepare(int tiles_x, int tiles_y, const BinsView& b, int64_t M, const double* md, int n_w,
                                double near_, double far_, const SplatRec* rec, int64_t* item_off, cudaStream_t st,
                                const ViewScratch* scr, bool q_ready, const Dyn* dyn, const int64_t* M_dev,
                                const int2* prect) {
  // dyn (sync-free): M is the capacity, M_dev the device count; item_off[M] (capacity index)
  // receives the pair total, nothing is read back (returns -1)
  const ViewScratch none{};
  const ViewScratch& sc = scr ? *scr : none;
  const int T = tiles_x * tiles_y;
  if (M <= 0) {
    cudaMemsetAsync(item_off, 0, sizeof(int64_t), st);
    return 0;
  }
  int32_t* widx = take_tmp(sc.widx, M, st);
  double* wz = take_tmp(sc.wz, M, st);
  int32_t* cnt = take_tmp(sc.cnt, M, st);
  int64_t* scratch = take_tmp(sc.scan, compact_blocks(M), st);
  const int* ovf = dyn ? dyn->ovf : nullptr;
  k_window_counts<<<T, 256, 0, st>>>(T, tiles_x, b.starts, b.items, b.nonmono, md, n_w, near_, far_, b.witems, rec,
                                     cnt, widx, wz, q_ready && sc.cnt, ovf, prect, b.cpos, b.clen);
  scan_counts(cnt, M, item_off, scratch, st, dyn ? M_dev : nullptr, ovf);
  if (dyn) {
    put_tmp(widx, sc.widx, st);
    put_tmp(wz, sc.wz, st);
    put_tmp(cnt, sc.cnt, st);
    put_tmp(scratch, sc.scan, st);
    return -1;
  }
  int64_t total = 0;
  cudaMemcpyAsync(&total, item_off + M, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  put_tmp(widx, sc.widx, st);
  put_tmp(wz, sc.wz, st);
  put_tmp(cnt, sc.cnt, st);
  put_tmp(scratch, sc.scan, st);
  cudaStreamSynchronize(st);
  return total;
}

void ts_impl_forward(int tiles_x, int tiles_y, const BinsView& b, const SplatRec* rec, const float* colors,
                     const Scene64& S64, int W, int H, double s, double t_stop, const int64_t* item_off,
                     int64_t n_pairs, uint32_t* pair_bits, float4* pair_rec, float* nmap, float* dmap, float* omap,
                     float* cmap, int32_t* n_proc, int32_t* n_blend, cudaStream_t st, const ViewScratch* scr,
                     const Dyn* dyn) {
  const int T = tiles_x * tiles_y;
  const int* ovf = dyn ? dyn->ovf : nullptr;
  int32_t* const given_order = scr ? scr->torder : nullptr;
  cudaMemsetAsync(pair_bits, 0, sizeof(uint32_t) * (size_t)TS_PAIR_BIT_WORDS(n_pairs), st);
  const int smem = (int)sizeof(FwdSmem);
  static const bool attr = [smem] {  // once (thread-safe static: lanes launch from several threads)
    cudaFuncSetAttribute(k_forward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_forward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)attr;
  int32_t* torder = take_tmp(given_order, T, st);
  k_tile_order<<<1, 1024, 0, st>>>(T, b.clen, torder);
  const bool clip_stops = (1.0 - kAlphaClipD) < t_stop;  // splat.py:14-15: T (1 - ALPHA_CLIP) < T_STOP
  if (colors && cmap)
    k_forward<true><<<T, TS_TILE_PX, smem, st>>>(torder, b.starts, b.cpos, b.witems, b.clen, rec, colors, S64, tiles_x,
                                                W, H, (float)s, s, (float)t_stop, clip_stops, item_off, pair_bits, pair_rec,
                                                nmap, dmap, omap, cmap, n_proc, n_blend, ovf);
  else
    k_forward<false><<<T, TS_TILE_PX, smem, st>>>(torder, b.starts, b.cpos, b.witems, b.clen, rec, nullptr, S64,
                                                 tiles_x, W, H, (float)s, s, (float)t_stop, clip_stops, item_off, pair_bits, pair_rec,
                                                 nmap, dmap, omap, nullptr, n_proc, n_blend, ovf);
  put_tmp(torder, given_order, st);
}

void ts_impl_backward(int tiles_x, int tiles_y, const BinsView& b, int64_t M, int64_t K, const SplatRec* rec,
                      const float* colors, const double* fsc, const int32_t* vert_ids, const int32_t* tet_ids,
                      const double* deform, int R, const Camera& cam, const int64_t* item_off,
                      const uint32_t* pair_bits, const float4* pair_rec, const float* maps[4],
                      const float* dmaps[4], const int32_t* n_proc, float* d_vert, float* d_color, cudaStream_t st,
                      const ViewScratch* scr, float* status, const int32_t* tiles, int n_tiles,
                      float* rows_out, const Dyn* dyn, const Fx* fx) {
  const int* ovf = dyn ? dyn->ovf : nullptr;
  const int T = tiles_x * tiles_y;
  if (M <= 0 || K <= 0) return;
  const int smem_c = (int)sizeof(BwdSmem<true>), smem = (int)sizeof(BwdSmem<false>);
  static const bool attr = [smem_c, smem] {  // once (thread-safe static)
    cudaFuncSetAttribute(k_backward<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_c);
    cudaFuncSetAttribute(k_backward<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_backward<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_c);
    cudaFuncSetAttribute(k_backward<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)attr;
  // rows_out: the plugin contract's per-splat gradients (backward_tiles, _core.pyx:344-471) —
  // the rows of the requested tiles are ADDED to rows_out and the vertex chain is not run
  float* const given_rows = rows_out ? rows_out : (scr ? scr->rows : nullptr);
  int32_t* const given_order = tiles ? const_cast<int32_t*>(tiles) : (scr ? scr->torder : nullptr);
  const int nblk = tiles ? n_tiles : T;
  if (nblk <= 0) return;
  const bool det = fx && fx->vert && !rows_out;  // fixed-point rows and outputs
  // per-splat rows: K <= M (fixed point: int64, twice the floats)
  float* rows = take_tmp(given_rows, (det ? 2 : 1) * kGr * (size_t)M, st);
  int32_t* torder = take_tmp(given_order, T, st);
  // the fused view path's workspace still holds this view's order from its forward
  if (!given_order) k_tile_order<<<1, 1024, 0, st>>>(T, b.clen, torder);
  const bool color = colors && maps[3] && dmaps[3] && (det ? fx->color != nullptr : (d_color || rows_out));
  if (!rows_out)
    cudaMemsetAsync(rows, 0,
                    (det ? 8 : 4) * (size_t)(color ? BwdSmem<true>::AS : BwdSmem<false>::AS) * (size_t)K, st);
  unsigned long long* bad = det ? fx->bad : nullptr;
#define TS_BWD_ARGS(C)                                                                                              \
  torder, b.starts, b.cpos, b.witems, b.clen, rec, C ? colors : nullptr, tiles_x, cam.width, cam.height,         \
      item_off, pair_bits, pair_rec, maps[0], maps[1], maps[2], C ? maps[3] : nullptr, dmaps[0], dmaps[1], dmaps[2], \
      C ? dmaps[3] : nullptr, n_proc, rows, status, ovf, bad
  if (color && det)
    k_backward<true, true><<<nblk, TS_TILE_PX, smem_c, st>>>(TS_BWD_ARGS(true));
  else if (color)
    k_backward<true, false><<<nblk, TS_TILE_PX, smem_c, st>>>(TS_BWD_ARGS(true));
  else if (det)
    k_backward<false, true><<<nblk, TS_TILE_PX, smem, st>>>(TS_BWD_ARGS(false));
  else
    k_backward<false, false><<<nblk, TS_TILE_PX, smem, st>>>(TS_BWD_ARGS(false));
#undef TS_BWD_ARGS
  if (rows_out) {
    put_tmp(torder, given_order, st);
    return;
  }
  int blocks = (int)((K + 127) / 128);
  if (blocks > 148 * 64) blocks = 148 * 64;
  const Fx fxa = det ? *fx : Fx{};
  const int64_t* Kd = dyn ? dyn->K : nullptr;
  if (color && det)
    k_chain<true, true><<<blocks, 128, 0, st>>>(K, rows, vert_ids, tet_ids, fsc, deform, make_grid(R), cam, nullptr,
                                                nullptr, Kd, ovf, fxa, rec);
  else if (color)
    k_chain<true, false><<<blocks, 128, 0, st>>>(K, rows, vert_ids, tet_ids, fsc, deform, make_grid(R), cam, d_vert,
                                                 d_color, Kd, ovf, fxa, rec);
  else if (det)
    k_chain<false, true><<<blocks, 128, 0, st>>>(K, rows, vert_ids, tet_ids, fsc, deform, make_grid(R), cam, nullptr,
                                                 nullptr, Kd, ovf, fxa, rec);
  else
    k_chain<false, false><<<blocks, 128, 0, st>>>(K, rows, vert_ids, tet_ids, fsc, deform, make_grid(R), cam, d_vert,
                                                  nullptr, Kd, ovf, fxa, rec);
  put_tmp(rows, given_rows, st);
  put_tmp(torder, given_order, st);
}

void ts_impl_list_flags(int T, const int64_t* starts, const int32_t* items, const double* md, double near_,
                        double far_, uint8_t* flags, cudaStream_t st) {
  if (T <= 0) return;
  k_list_flags<<<(T + 7) / 8, 256, 0, st>>>(T, starts, items, md, near_, far_, flags);
}

void ts_impl_saved_records(const int32_t* tiles, int n_tiles, int tiles_x, int W, int H, const BinsView& b,
                           const SplatRec* rec, const int64_t* item_off, const uint32_t* pair_bits,
                           const float4* pair_rec, const int32_t* n_proc, const int64_t* rec_off, int64_t* idx,
                           double* alpha, cudaStream_t st) {
  if (n_tiles <= 0) return;
  k_saved_records<<<n_tiles, TS_TILE_PX, 0, st>>>(tiles, tiles_x, W, H, b.starts, b.cpos, b.witems, b.clen, rec,
                                                  item_off, pair_bits, pair_rec, n_proc, rec_off, idx, alpha);
}

void ts_impl_hist(unsigned long long out[32], int reset) {
  cudaMemcpyFromSymbol(out, g_ts_hist, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(g_ts_hist, z, sizeof(z));
  }
}

void ts_impl_counters(unsigned long long out[8], int reset) {
  cudaMemcpyFromSymbol(out, g_ts_counters, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_ts_counters, z, sizeof(z));
  }
}

void ts_impl_phases(unsigned long long out[16], int reset) {
  cudaMemcpyFromSymbol(out, g_ts_phase, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_ts_phase, z, sizeof(z));
  }
}

void ts_impl_debug_flags(int flags) {
  h_debug_flags = flags;
  cudaMemcpyToSymbol(g_ts_debug_flags, &flags, sizeof(int));
}

void ts_impl_tile_times(unsigned long long* t2, unsigned int* sm, int n) {
  cudaMemcpyFromSymbol(t2, g_ts_tile_time, sizeof(unsigned long long) * 2 * n);
  cudaMemcpyFromSymbol(sm, g_ts_tile_sm, sizeof(unsigned int) * n);
}
