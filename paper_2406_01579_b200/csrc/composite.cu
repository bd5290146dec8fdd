// composite.cu — K6 forward compositing, K7 backward + vertex chain, N_w window.
//
// Forward (replaces forward_tiles, _core.pyx:98-229): one 256-thread CTA per 16x16 tile,
// one pixel per thread.  The tile's list is staged through shared memory in chunks; each
// staged record carries the four projected faces as sign-normalised edge functions in
// splat-anchored FP32 coordinates.  Inside/outside decisions that fall within a rigorous
// FP32 error band of an edge are recomputed with the reference's exact FP64 arithmetic
// (records.cuh: splat_hits_exact), so the set of blended (pixel, splat) pairs matches the
// FP64 reference; the blend itself is FP32.  A CTA leaves its loop as soon as every pixel
// has reached T < t_stop (__syncthreads_and = block-wide ballot).
//
// The N_w resorting window (_core.pyx:171-187) pops, for every pixel of a tile, the same
// sequence — it depends only on the tile list, never on the pixel.  When mean depth is
// non-decreasing along the list (bin.cu flags it), the window is the identity; otherwise
// k_window replays the reference's window once per tile into witems.
//
// Backward (replaces backward_tiles _core.pyx:344-471 + splat_grads_to_vertices
// raster.py:253-306): the same CTA/pixel layout walks the list FRONT to back.  The
// reference's suffix sums are C_final - prefix (C_final = the forward maps), and the
// d_alpha * d(alpha)/d(f) product is formed as g.(T x (1-a) - suffix) * s * sigmoid, which
// is the reference's expression with the (1-a) factor cancelled algebraically (no
// division by 1-a, no reverse walk, no per-pixel record lists).  Per (tile, splat) the
// 23 gradient scalars are reduced across the warp with a transposed butterfly (31
// shuffles), across warps with shared-memory atomics, and written to a per-pair row;
// k_chain gathers each splat's rows in a fixed order (deterministic, atomic-free) and
// applies the normal chain and the camera chain in FP64, then scatters to vertices with
// one red.global.add.v4.f32 per (splat, vertex).
#include "internal.cuh"

namespace ts {

constexpr float kAlphaClipF = 0.9999f;  // splat.py:14
constexpr float kOneMinusClipF = 1e-4f;
constexpr int kChF = 128;  // forward chunk (records per shared-memory stage)
constexpr int kChB = 64;   // backward chunk
constexpr int kGr = 24;    // floats per (tile, splat) gradient row

struct __align__(16) Staged {
  int rx0, rx1, ry0, ry1;
  float band;
  uint32_t flags;
  int k;
  float md;
  float iz[4], df[4];  // 1/z; f_i - f_0
  float eux[4], euy[4], cu[4], evx[4], evy[4], cv[4], adet[4];
  float n[3];
  float fband;  // 3 * band * (z_max / z_min) * max|f|: FP32 f_hit error = fband / |det_face|
  float ftol0;  // rounding of the stored f deltas
  float f0;
  float pad[2];
};
static_assert(sizeof(Staged) == 208, "Staged must be 208 bytes");

// diagnostics: [0] pairs re-decided in FP64 because of an edge / degenerate face,
// [1] pairs re-decided in FP64 because of an alpha threshold
__device__ unsigned long long g_ts_counters[4];

__device__ __forceinline__ void stage(const SplatRec* __restrict__ recs, int k, Staged& s) {
  const float4* p = reinterpret_cast<const float4*>(recs + k);
  float4 q0 = __ldg(p + 0), q1 = __ldg(p + 1), q2 = __ldg(p + 2), q3 = __ldg(p + 3), q4 = __ldg(p + 4),
         q5 = __ldg(p + 5);
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
  s.f0 = q4.x; s.df[0] = 0.f; s.df[1] = q4.y; s.df[2] = q4.z; s.df[3] = q4.w;
  s.n[0] = q5.x; s.n[1] = q5.y; s.n[2] = q5.z;
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
  }
  // error bound of FP32 f_hit: edge-function error (band/16) over |det|, times depth ratio
  // FP32 f_hit - f_0 = sum(lambda_i df_i): error <= 0.375 band zr / |det| * spread per face
  float fmax = fmaxf(fabsf(s.df[1]), fmaxf(fabsf(s.df[2]), fabsf(s.df[3])));
  float izmin = fminf(fminf(s.iz[0], s.iz[1]), fminf(s.iz[2], s.iz[3]));
  float izmax = fmaxf(fmaxf(s.iz[0], s.iz[1]), fmaxf(s.iz[2], s.iz[3]));
  s.fband = 0.75f * s.band * (izmax / izmin) * fmax;
  s.ftol0 = 1e-6f * fmax;
}

struct Hit {
  float fp, fn;
  int fip, fin;
};

// 0: no hit, 1: hit, 2: undecided in FP32 (caller takes the exact FP64 path)
__device__ __forceinline__ int eval_hits(const Staged& s, float px, float py, Hit& h) {
  if (s.flags & 16u) return 2;
  const float band = s.band;
  int nh = 0, lo = -1, hi = -1;
  float zlo = 0.f, zhi = 0.f, flo = 0.f, fhi = 0.f;
#pragma unroll
  for (int fi = 0; fi < 4; ++fi) {
    if (!((s.flags >> fi) & 1u)) continue;
    float u = fmaf(s.eux[fi], px, fmaf(s.euy[fi], py, s.cu[fi]));
    float v = fmaf(s.evx[fi], px, fmaf(s.evy[fi], py, s.cv[fi]));
    float w = s.adet[fi] - u - v;
    if (u < -band || v < -band || w < -band) continue;
    if (u <= band || v <= band || w <= band) return 2;
    const int ia = face_vert(fi, 0), ib = face_vert(fi, 1), ic = face_vert(fi, 2);
    float wa = w * s.iz[ia], wb = u * s.iz[ib], wc = v * s.iz[ic];
    float D = wa + wb + wc;
    float rD = 1.0f / D;
    float zp = s.adet[fi] * rD;
    float fh = (wa * s.df[ia] + wb * s.df[ib] + wc * s.df[ic]) * rD;  // f_hit - f0
    if (nh == 0) {
      zlo = zhi = zp; flo = fhi = fh; lo = hi = fi;
    } else {
      if (zp < zlo) { zlo = zp; flo = fh; lo = fi; }
      if (zp > zhi) { zhi = zp; fhi = fh; hi = fi; }
    }
    ++nh;
  }
  if (nh < 2) return 0;
  h.fp = flo; h.fn = fhi; h.fip = lo; h.fin = hi;
  return 1;
}

__device__ __forceinline__ float softplus_tail(float x) { return log1pf(expf(-fabsf(x))); }

// Outcome of one (pixel, splat) pair: whether it blends, and the values the blend uses.
struct Blend {
  float fp, fn;  // SDF at entry / exit
  int fip, fin;  // entry / exit faces
  float a, om;   // clipped alpha and 1 - alpha
  bool clipped;  // alpha_un > ALPHA_CLIP (no d_alpha/d_f, _core.pyx:462)
};

// Exact replica of the reference decision chain in FP64 (_core.pyx:67-95, 35-36, 190-196).
__device__ __noinline__ bool blend_exact(const Scene64& S, int k, int xi, int yi, double s, Blend& b) {
  double fp, fn;
  int i0, i1;
  if (!splat_hits_exact(S, k, xi + 0.5, yi + 0.5, fp, fn, i0, i1)) return false;
  double d = dsub(softplus_d(dmul(-s, fp)), softplus_d(dmul(-s, fn)));
  double a = dsub(1.0, exp(d));
  if (a <= 0.0) return false;
  b.fp = (float)fp;
  b.fn = (float)fn;
  b.fip = i0;
  b.fin = i1;
  b.clipped = a > 1.0 - 1e-4;
  if (b.clipped) {
    b.a = kAlphaClipF;
    b.om = kOneMinusClipF;
  } else {
    b.a = (float)a;
    b.om = (float)exp(d);
  }
  return true;
}

// FP32 fast path with error-bounded decisions; anything within the bounds of a decision
// threshold (face edges, alpha == 0, alpha == ALPHA_CLIP, FP32 underflow) is re-decided
// by blend_exact so the blended set matches the FP64 reference.
__device__ __forceinline__ bool blend_of(const Staged& r, float px, float py, int xi, int yi, float s, double s64,
                                         const Scene64& S, Blend& b) {
  Hit h;  // h.fp / h.fn are f - f0 here
  const int e = eval_hits(r, px, py, h);
  if (e == 0) return false;
  if (e == 1) {
    const float dfl = h.fp - h.fn;  // f_prev - f_next, f0 cancels exactly
    const float ftol = r.fband / fminf(r.adet[h.fip], r.adet[h.fin]) + r.ftol0;
    if (dfl < -ftol) return false;  // f_prev < f_next: alpha <= 0 exactly
    if (dfl > ftol) {
      const float fp = r.f0 + h.fp, fn = r.f0 + h.fn;
      const float x = -s * fp, y = -s * fn;
      float d;
      if (x > 0.f && y > 0.f)
        d = -s * dfl + (softplus_tail(x) - softplus_tail(y));
      else
        d = (fmaxf(x, 0.f) + softplus_tail(x)) - (fmaxf(y, 0.f) + softplus_tail(y));
      const float a_un = -expm1f(d);
      // alpha > 1e-10 and not at the clip threshold: the FP64 reference decides the same
      if (d < -1e-10f && fabsf(a_un - kAlphaClipF) > 2e-6f) {
        b.fp = fp;
        b.fn = fn;
        b.fip = h.fip;
        b.fin = h.fin;
        b.clipped = a_un > kAlphaClipF;
        if (b.clipped) {
          b.a = kAlphaClipF;
          b.om = kOneMinusClipF;
        } else {
          b.a = a_un;
          b.om = expf(d);
        }
        return true;
      }
    }
    atomicAdd(&g_ts_counters[1], 1ull);
  } else {
    atomicAdd(&g_ts_counters[0], 1ull);
  }
  return blend_exact(S, r.k, xi, yi, s64, b);
}

__device__ __forceinline__ float sigmoidf_stable(float x) {
  if (x >= 0.f) return 1.0f / (1.0f + expf(-x));
  float e = expf(x);
  return e / (1.0f + e);
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

template <bool COLOR>
__global__ void __launch_bounds__(TS_TILE_PX) k_forward(
    const int64_t* __restrict__ starts, const int32_t* __restrict__ items, const int32_t* __restrict__ witems,
    const uint8_t* __restrict__ nonmono, const SplatRec* __restrict__ recs, const float* __restrict__ colors,
    Scene64 S64, int tiles_x, int W, int H, float s, double s64, float t_stop, float* __restrict__ normal_map,
    float* __restrict__ depth_map, float* __restrict__ opacity_map, float* __restrict__ color_map,
    int32_t* __restrict__ n_proc, int32_t* __restrict__ n_blend) {
  __shared__ Staged sh[kChF];
  __shared__ float shc[COLOR ? kChF : 1][3];
  const int tile = blockIdx.x;
  const int xi = (tile % tiles_x) * TS_TILE + (threadIdx.x & (TS_TILE - 1));
  const int yi = (tile / tiles_x) * TS_TILE + (threadIdx.x / TS_TILE);
  const bool inside = xi < W && yi < H;
  const int64_t lo = starts[tile];
  const int L = (int)(starts[tile + 1] - lo);
  const int32_t* list = (nonmono[tile] ? witems : items) + lo;
  float T = 1.f;
  Accum<COLOR> acc;
  acc.zero();
  unsigned nbbox = 0;  // pairs passing the pixel-rect test (roofline work model)
  bool done = !inside;
  int nproc = inside ? L : 0, nb = 0;
  for (int base = 0; base < L; base += kChF) {
    const int n = min(kChF, L - base);
    if (threadIdx.x < n) {
      int k = list[base + threadIdx.x];
      stage(recs, k, sh[threadIdx.x]);
      if (COLOR)
        for (int c = 0; c < 3; ++c) shc[threadIdx.x][c] = colors[(int64_t)k * 3 + c];
    }
    __syncthreads();
    if (!done) {
      for (int j = 0; j < n; ++j) {
        const Staged& r = sh[j];
        if (xi < r.rx0 || xi > r.rx1 || yi < r.ry0 || yi > r.ry1) continue;
        ++nbbox;
        const float px = (float)(xi - r.rx0) + 0.5f, py = (float)(yi - r.ry0) + 0.5f;
        Blend bl;
        if (!blend_of(r, px, py, xi, yi, s, s64, S64, bl)) continue;
        acc.add(__fmul_rn(T, bl.a), r, COLOR ? shc[j] : nullptr);
        T = __fmul_rn(T, bl.om);
        ++nb;
        if (T < t_stop) {
          done = true;
          nproc = base + j + 1;
          break;
        }
      }
    }
    if (__syncthreads_and(done)) break;
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
  const unsigned wb = warp_sum(nbbox);
  if ((threadIdx.x & 31) == 0 && wb) atomicAdd(&g_ts_counters[2], (unsigned long long)wb);
}

// per-tile replay of the reference window (_core.pyx:171-187) for tiles whose list is
// not mean-depth monotone; one thread per flagged tile, window state in global scratch
__global__ void k_window(int T, const int64_t* __restrict__ starts, const int32_t* __restrict__ items,
                         const uint8_t* __restrict__ nonmono, const double* __restrict__ md, int n_w,
                         int32_t* __restrict__ witems, int32_t* __restrict__ widx_s, double* __restrict__ wz_s) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T || !nonmono[t]) return;
  const int64_t lo = starts[t], L = starts[t + 1] - lo;
  int32_t* widx = widx_s + lo;
  double* wz = wz_s + lo;
  int64_t wcount = 0, pos = 0, out = 0;
  for (;;) {
    while (wcount < n_w && pos < L) {
      int32_t k = items[lo + pos];
      widx[wcount] = k;
      wz[wcount] = md[k];
      ++wcount;
      ++pos;
    }
    if (wcount == 0) break;
    int64_t m = 0;
    for (int64_t i = 1; i < wcount; ++i)
      if (wz[i] < wz[m]) m = i;
    witems[lo + out++] = widx[m];
    for (int64_t i = m; i < wcount - 1; ++i) {
      widx[i] = widx[i + 1];
      wz[i] = wz[i + 1];
    }
    --wcount;
  }
}

// backward of one face hit (_core.pyx:295-341) into per-vertex rows gr[0..15]
template <int FI>
__device__ __forceinline__ void face_bwd(const Staged& r, float px, float py, float g, float* gr) {
  constexpr int ia = face_vert(FI, 0), ib = face_vert(FI, 1), ic = face_vert(FI, 2);
  const float inv_ad = 1.0f / r.adet[FI];
  float u = fmaf(r.eux[FI], px, fmaf(r.euy[FI], py, r.cu[FI])) * inv_ad;
  float v = fmaf(r.evx[FI], px, fmaf(r.evy[FI], py, r.cv[FI])) * inv_ad;
  float wbar = 1.0f - u - v;
  float w0 = wbar * r.iz[ia], w1 = u * r.iz[ib], w2 = v * r.iz[ic];
  float iS = 1.0f / (w0 + w1 + w2);
  float fh = (w0 * r.df[ia] + w1 * r.df[ib] + w2 * r.df[ic]) * iS;  // f_hit - f0
  gr[ia] += g * w0 * iS;
  gr[ib] += g * w1 * iS;
  gr[ic] += g * w2 * iS;
  float dw0 = g * (r.df[ia] - fh) * iS, dw1 = g * (r.df[ib] - fh) * iS, dw2 = g * (r.df[ic] - fh) * iS;
  gr[4 + ia] += dw0 * (-w0 * r.iz[ia]);
  gr[4 + ib] += dw1 * (-w1 * r.iz[ib]);
  gr[4 + ic] += dw2 * (-w2 * r.iz[ic]);
  float gu = -dw0 * r.iz[ia] + dw1 * r.iz[ib];
  float gv = -dw0 * r.iz[ia] + dw2 * r.iz[ic];
  float qx = (r.eux[FI] * gu + r.evx[FI] * gv) * inv_ad;
  float qy = (r.euy[FI] * gu + r.evy[FI] * gv) * inv_ad;
  gr[8 + ia] -= qx * wbar;
  gr[12 + ia] -= qy * wbar;
  gr[8 + ib] -= qx * u;
  gr[12 + ib] -= qy * u;
  gr[8 + ic] -= qx * v;
  gr[12 + ic] -= qy * v;
}

// lane L ends with the warp total of value L (transposed butterfly, 31 shuffles)
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32]) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      float send = up ? v[i] : v[i + h];
      float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

template <bool COLOR>
__global__ void __launch_bounds__(TS_TILE_PX) k_backward(
    const int64_t* __restrict__ starts, const int32_t* __restrict__ items, const int32_t* __restrict__ witems,
    const uint8_t* __restrict__ nonmono, const SplatRec* __restrict__ recs, const float* __restrict__ colors,
    Scene64 S64, int tiles_x, int W, int H, float s, double s64, const float* __restrict__ normal_map,
    const float* __restrict__ depth_map, const float* __restrict__ opacity_map, const float* __restrict__ color_map,
    const float* __restrict__ d_normal, const float* __restrict__ d_depth, const float* __restrict__ d_opacity,
    const float* __restrict__ d_color, const int32_t* __restrict__ n_proc, float* __restrict__ rows) {
  __shared__ Staged sh[kChB];
  __shared__ float acc_s[kChB][kGr];
  __shared__ float shc[COLOR ? kChB : 1][3];
  __shared__ int maxproc_s;
  const int tile = blockIdx.x;
  const int xi = (tile % tiles_x) * TS_TILE + (threadIdx.x & (TS_TILE - 1));
  const int yi = (tile / tiles_x) * TS_TILE + (threadIdx.x / TS_TILE);
  const bool inside = xi < W && yi < H;
  const int64_t lo = starts[tile];
  const int L = (int)(starts[tile + 1] - lo);
  const int32_t* list = (nonmono[tile] ? witems : items) + lo;
  const int64_t p = inside ? (int64_t)yi * W + xi : 0;
  const int nproc = inside ? n_proc[p] : 0;
  if (threadIdx.x == 0) maxproc_s = 0;
  __syncthreads();
  if (nproc > 0) atomicMax(&maxproc_s, nproc);
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
  __syncthreads();
  const int maxproc = maxproc_s;
  float T = 1.f;
  Accum<COLOR> P;
  P.zero();
  for (int base = 0; base < maxproc; base += kChB) {
    const int n = min(kChB, maxproc - base);
    if (threadIdx.x < n) {
      int k = list[base + threadIdx.x];
      stage(recs, k, sh[threadIdx.x]);
      if (COLOR)
        for (int c = 0; c < 3; ++c) shc[threadIdx.x][c] = colors[(int64_t)k * 3 + c];
    }
    for (int i = threadIdx.x; i < n * kGr; i += TS_TILE_PX) (&acc_s[0][0])[i] = 0.f;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const Staged& r = sh[j];
      float gr[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) gr[i] = 0.f;
      bool contrib = false;
      if (base + j < nproc && xi >= r.rx0 && xi <= r.rx1 && yi >= r.ry0 && yi <= r.ry1) {
        const float px = (float)(xi - r.rx0) + 0.5f, py = (float)(yi - r.ry0) + 0.5f;
        Blend bl;
        if (blend_of(r, px, py, xi, yi, s, s64, S64, bl)) {
          contrib = true;
          const float* col = COLOR ? shc[j] : nullptr;
          const float w = __fmul_rn(T, bl.a);
          P.add(w, r, col);
          gr[19] = g_d * w;
          gr[16] = g_n[0] * w;
          gr[17] = g_n[1] * w;
          gr[18] = g_n[2] * w;
          if (COLOR) {
            gr[20] = g_c[0] * w;
            gr[21] = g_c[1] * w;
            gr[22] = g_c[2] * w;
          }
          if (!bl.clipped) {
            const float Tom = T * bl.om;
            float G = g_o * (Tom - (C_o - P.o)) + g_d * (Tom * r.md - (C_d - P.d));
#pragma unroll
            for (int i = 0; i < 3; ++i) G += g_n[i] * (Tom * r.n[i] - (C_n[i] - P.n[i]));
            if (COLOR)
#pragma unroll
              for (int i = 0; i < 3; ++i) G += g_c[i] * (Tom * col[i] - (C_c[i] - P.c[i]));
            const float dfp = G * s * sigmoidf_stable(-s * bl.fp);
            const float dfn = -G * s * sigmoidf_stable(-s * bl.fn);
            const float g0 = (bl.fip == 0 ? dfp : 0.f) + (bl.fin == 0 ? dfn : 0.f);
            const float g1 = (bl.fip == 1 ? dfp : 0.f) + (bl.fin == 1 ? dfn : 0.f);
            const float g2 = (bl.fip == 2 ? dfp : 0.f) + (bl.fin == 2 ? dfn : 0.f);
            const float g3 = (bl.fip == 3 ? dfp : 0.f) + (bl.fin == 3 ? dfn : 0.f);
            if (bl.fip == 0 || bl.fin == 0) face_bwd<0>(r, px, py, g0, gr);
            if (bl.fip == 1 || bl.fin == 1) face_bwd<1>(r, px, py, g1, gr);
            if (bl.fip == 2 || bl.fin == 2) face_bwd<2>(r, px, py, g2, gr);
            if (bl.fip == 3 || bl.fin == 3) face_bwd<3>(r, px, py, g3, gr);
          }
          T = __fmul_rn(T, bl.om);
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        float tot = warp_transpose_reduce(gr);
        const int lane = threadIdx.x & 31;
        if (lane < (COLOR ? 23 : 20)) atomicAdd(&acc_s[j][lane], tot);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += TS_TILE_PX) {
      float4* dst = reinterpret_cast<float4*>(rows + (lo + base + t) * kGr);
      const float4* src = reinterpret_cast<const float4*>(&acc_s[t][0]);
#pragma unroll
      for (int i = 0; i < kGr / 4; ++i) dst[i] = src[i];
    }
    __syncthreads();
  }
  // positions no pixel reached: zero rows so the gather sees every pair
  for (int64_t q = maxproc + threadIdx.x; q < L; q += TS_TILE_PX) {
    float4* dst = reinterpret_cast<float4*>(rows + (lo + q) * kGr);
#pragma unroll
    for (int i = 0; i < kGr / 4; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// per-splat gather + normal chain + camera chain (raster.py:253-306), FP64 math
template <bool COLOR>
__global__ void k_chain(int64_t K, const int64_t* __restrict__ splat_off, const int32_t* __restrict__ pos_of,
                        const float* __restrict__ rows, const int32_t* __restrict__ vert_ids,
                        const int32_t* __restrict__ tet_ids, const double* __restrict__ fsc,
                        const double* __restrict__ deform, Grid G, Camera cam, float* __restrict__ d_vert,
                        float* __restrict__ d_color) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    float a[kGr];
#pragma unroll
    for (int i = 0; i < kGr; ++i) a[i] = 0.f;
    for (int64_t r = splat_off[k]; r < splat_off[k + 1]; ++r) {
      const float4* src = reinterpret_cast<const float4*>(rows + (int64_t)pos_of[r] * kGr);
#pragma unroll
      for (int i = 0; i < kGr / 4; ++i) {
        float4 q = __ldg(src + i);
        a[4 * i] += q.x; a[4 * i + 1] += q.y; a[4 * i + 2] += q.z; a[4 * i + 3] += q.w;
      }
    }
    double dF[4], dZ[4], dPx[4], dPy[4], dPos[4][3];
    const double dMd = a[19];
    for (int v = 0; v < 4; ++v) {
      dF[v] = a[v];
      dZ[v] = (double)a[4 + v] + dMd / 4.0;
      dPx[v] = a[8 + v];
      dPy[v] = a[12 + v];
      dPos[v][0] = dPos[v][1] = dPos[v][2] = 0.0;
    }
    uint32_t vid[4];
    double P[4][3], f[4];
    for (int v = 0; v < 4; ++v) {
      vid[v] = (uint32_t)vert_ids[k * 4 + v];
      vertex_position(vid[v], G, deform, P[v]);
      f[v] = fsc[k * 4 + v];
    }
    // normal chain: n = g/|g|, dL/dg = (I - n n^T) dL/dn / |g|, dL/df = B^-T [dL/dg, 0]
    double g[3], c1[3], c2[3], c3[3];
    double det = tet_gradient(P, f, g, c1, c2, c3);
    double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (gn >= 1e-8 && det != 0.0) {
      double n[3] = {g[0] / gn, g[1] / gn, g[2] / gn};
      double dn[3] = {a[16], a[17], a[18]};
      double dot = n[0] * dn[0] + n[1] * dn[1] + n[2] * dn[2];
      double dg[3];
      for (int i = 0; i < 3; ++i) dg[i] = (dn[i] - n[i] * dot) / gn;
      double d1 = (c1[0] * dg[0] + c1[1] * dg[1] + c1[2] * dg[2]) / det;
      double d2 = (c2[0] * dg[0] + c2[1] * dg[1] + c2[2] * dg[2]) / det;
      double d3 = (c3[0] * dg[0] + c3[1] * dg[1] + c3[2] * dg[2]) / det;
      double dfn[4] = {-(d1 + d2 + d3), d1, d2, d3};
      for (int v = 0; v < 4; ++v) {
        dF[v] += dfn[v];
        for (int i = 0; i < 3; ++i) dPos[v][i] -= dfn[v] * g[i];
      }
    }
    // camera chain: pixel = (fx X/Z + cx, fy Y/Z + cy), depth = Z
    for (int v = 0; v < 4; ++v) {
      double pc[3];
      for (int r = 0; r < 3; ++r)
        pc[r] = P[v][0] * cam.R[r * 3] + P[v][1] * cam.R[r * 3 + 1] + P[v][2] * cam.R[r * 3 + 2] + cam.t[r];
      const double X = pc[0], Y = pc[1], Z = pc[2];
      const double dpc[3] = {dPx[v] * cam.fx / Z, dPy[v] * cam.fy / Z,
                             -dPx[v] * cam.fx * X / (Z * Z) - dPy[v] * cam.fy * Y / (Z * Z) + dZ[v]};
      for (int j = 0; j < 3; ++j)
        dPos[v][j] += dpc[0] * cam.R[j] + dpc[1] * cam.R[3 + j] + dpc[2] * cam.R[6 + j];
      red_add_v4(d_vert + (size_t)vid[v] * 4, (float)dF[v], (float)dPos[v][0], (float)dPos[v][1], (float)dPos[v][2]);
    }
    if (COLOR) {
      const int64_t t = tet_ids[k];
      for (int c = 0; c < 3; ++c) atomicAdd(d_color + t * 3 + c, a[20 + c]);
    }
  }
}

}  // namespace ts

using namespace ts;


void ts_impl_window(int T, const BinsView& b, int64_t M, const double* md, int n_w, cudaStream_t st) {
  if (M <= 0) return;
  int32_t* widx = nullptr;
  double* wz = nullptr;
  cudaMallocAsync(&widx, sizeof(int32_t) * M, st);
  cudaMallocAsync(&wz, sizeof(double) * M, st);
  k_window<<<(T + 63) / 64, 64, 0, st>>>(T, b.starts, b.items, b.nonmono, md, n_w, b.witems, widx, wz);
  cudaFreeAsync(widx, st);
  cudaFreeAsync(wz, st);
}

void ts_impl_forward(int tiles_x, int tiles_y, const BinsView& b, const SplatRec* rec, const float* colors,
                     const Scene64& S64, int W, int H, double s, float t_stop, float* nmap, float* dmap, float* omap,
                     float* cmap, int32_t* n_proc, int32_t* n_blend, cudaStream_t st) {
  const int T = tiles_x * tiles_y;
  if (colors && cmap)
    k_forward<true><<<T, TS_TILE_PX, 0, st>>>(b.starts, b.items, b.witems, b.nonmono, rec, colors, S64, tiles_x, W,
                                             H, (float)s, s, t_stop, nmap, dmap, omap, cmap, n_proc, n_blend);
  else
    k_forward<false><<<T, TS_TILE_PX, 0, st>>>(b.starts, b.items, b.witems, b.nonmono, rec, nullptr, S64, tiles_x,
                                              W, H, (float)s, s, t_stop, nmap, dmap, omap, nullptr, n_proc, n_blend);
}

void ts_impl_backward(int tiles_x, int tiles_y, const BinsView& b, int64_t M, int64_t K, const SplatRec* rec,
                      const float* colors, const Scene64& S64, const int32_t* vert_ids, const int32_t* tet_ids,
                      const double* deform, int R, const Camera& cam, double s, const float* maps[4],
                      const float* dmaps[4], const int32_t* n_proc, float* d_vert, float* d_color,
                      cudaStream_t st) {
  const int T = tiles_x * tiles_y;
  if (M <= 0 || K <= 0) return;
  float* rows = nullptr;
  cudaMallocAsync(&rows, sizeof(float) * kGr * (size_t)M, st);
  const bool color = colors && maps[3] && dmaps[3] && d_color;
  if (color)
    k_backward<true><<<T, TS_TILE_PX, 0, st>>>(b.starts, b.items, b.witems, b.nonmono, rec, colors, S64, tiles_x,
                                              cam.width, cam.height, (float)s, s, maps[0], maps[1], maps[2], maps[3],
                                              dmaps[0], dmaps[1], dmaps[2], dmaps[3], n_proc, rows);
  else
    k_backward<false><<<T, TS_TILE_PX, 0, st>>>(b.starts, b.items, b.witems, b.nonmono, rec, nullptr, S64, tiles_x,
                                               cam.width, cam.height, (float)s, s, maps[0], maps[1], maps[2], nullptr,
                                               dmaps[0], dmaps[1], dmaps[2], nullptr, n_proc, rows);
  int blocks = (int)((K + 127) / 128);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (color)
    k_chain<true><<<blocks, 128, 0, st>>>(K, b.splat_off, b.pos_of, rows, vert_ids, tet_ids, S64.f, deform, make_grid(R), cam,
                                          d_vert, d_color);
  else
    k_chain<false><<<blocks, 128, 0, st>>>(K, b.splat_off, b.pos_of, rows, vert_ids, tet_ids, S64.f, deform, make_grid(R),
                                           cam, d_vert, nullptr);
  cudaFreeAsync(rows, st);
}

void ts_impl_counters(unsigned long long out[4], int reset) {
  cudaMemcpyFromSymbol(out, g_ts_counters, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_ts_counters, z, sizeof(z));
  }
}
