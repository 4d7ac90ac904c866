// Fused single-pass elementwise kernels (reference: pkg/src/fuseq/kernels.py).
//
// Numerics follow SURVEY.md Appendix A (the numba-inferred types of the
// reference kernels): f64 statistics for layer norm and softmax, fp32
// two-rounding affine epilogues (no FMA contraction: __fmul_rn/__fadd_rn),
// f64 erf for GELU. Reductions are warp/block trees in a fixed order, so the
// results are deterministic run to run (the reference is deterministic too).
//
// All are HBM-bound: algorithmic bytes = inputs read + outputs written.
#include "fq_common.cuh"

namespace fq {

// fp16 copy of 4 outputs (the next GEMM's operand): hi only (throughput mode)
// or the exact mode's hi + lo pair (split_xh) when lo != NULL.
__device__ __forceinline__ void store_half4(h16* hi, h16* lo, int64_t off, float4 o) {
  uint2 ph, pl;
  split_xh2(o.x, o.y, ph.x, pl.x);
  split_xh2(o.z, o.w, ph.y, pl.y);
  *reinterpret_cast<uint2*>(hi + off) = ph;
  if (lo) *reinterpret_cast<uint2*>(lo + off) = pl;
}

// ---------------------------------------------------------------------------
// layer norm / bias+residual+layer norm: one CTA per row, the row staged in
// shared memory so the three sweeps of kernels.py:22-35 read HBM once.
// ---------------------------------------------------------------------------
template <bool kBiasRes>
__global__ void __launch_bounds__(256) layer_norm_kernel(
    const float* __restrict__ x, int64_t ldx, const float* __restrict__ bias,
    const float* __restrict__ res, int64_t ldr, const float* __restrict__ gamma,
    const float* __restrict__ beta, double eps, int d, float* __restrict__ out, int64_t ldo,
    h16* __restrict__ out16, h16* __restrict__ out16lo, int64_t ldo16) {
  pdl_enter();
  extern __shared__ float srow[];
  __shared__ double red[8];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * ldx;
  double s = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float u = xr[j];
    if (kBiasRes) u = fadd_rn(fadd_rn(u, bias[j]), res[row * ldr + j]);  // kernels.py:64
    srow[j] = u;
    s += (double)u;
  }
  const double mean = block_sum(s, red) / d;
  double v = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double t = (double)srow[j] - mean;
    v += t * t;
  }
  const double inv = 1.0 / sqrt(block_sum(v, red) / d + eps);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float n = (float)(((double)srow[j] - mean) * inv);
    float o = fadd_rn(fmul_rn(n, gamma[j]), beta[j]);  // kernels.py:35
    if (out) out[row * ldo + j] = o;
    if (out16) {
      if (out16lo) split_xh(o, out16[row * ldo16 + j], out16lo[row * ldo16 + j]);
      else out16[row * ldo16 + j] = f2h(o);
    }
  }
}

// Warp-per-row variant for d % 128 == 0, d <= 128 * kMaxV: the row lives in
// registers (float4 per lane per 128 columns), statistics reduce with f64
// shuffles — one HBM read, no shared memory, no block barriers.
constexpr int kMaxV = 8;  // d <= 1024 (wider rows use the CTA kernel)
template <bool kBiasRes>
__global__ void __launch_bounds__(256) layer_norm_warp_kernel(
    const float* __restrict__ x, int64_t ldx, const float* __restrict__ bias,
    const float* __restrict__ res, int64_t ldr, const float* __restrict__ gamma,
    const float* __restrict__ beta, double eps, int64_t rows, int d, float* __restrict__ out,
    int64_t ldo, h16* __restrict__ out16, h16* __restrict__ out16lo, int64_t ldo16) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= rows) return;
  const int nv = d >> 7;
  float4 u[kMaxV];
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kMaxV; ++i) {
    if (i < nv) {
      const int c = (i * 32 + lane) * 4;
      float4 a = *reinterpret_cast<const float4*>(x + row * ldx + c);
      if (kBiasRes) {
        float4 b = *reinterpret_cast<const float4*>(bias + c);
        float4 r = *reinterpret_cast<const float4*>(res + row * ldr + c);
        a.x = fadd_rn(fadd_rn(a.x, b.x), r.x);  // kernels.py:64 summand
        a.y = fadd_rn(fadd_rn(a.y, b.y), r.y);
        a.z = fadd_rn(fadd_rn(a.z, b.z), r.z);
        a.w = fadd_rn(fadd_rn(a.w, b.w), r.w);
      }
      u[i] = a;
      s += ((double)a.x + (double)a.y) + ((double)a.z + (double)a.w);
    }
  }
  const double mean = warp_sum(s) / d;
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < kMaxV; ++i) {
    if (i < nv) {
      double t0 = u[i].x - mean, t1 = u[i].y - mean, t2 = u[i].z - mean, t3 = u[i].w - mean;
      v += (t0 * t0 + t1 * t1) + (t2 * t2 + t3 * t3);
    }
  }
  const double inv = 1.0 / sqrt(warp_sum(v) / d + eps);
#pragma unroll
  for (int i = 0; i < kMaxV; ++i) {
    if (i < nv) {
      const int c = (i * 32 + lane) * 4;
      const float4 g = *reinterpret_cast<const float4*>(gamma + c);
      const float4 bb = *reinterpret_cast<const float4*>(beta + c);
      float4 o;
      o.x = fadd_rn(fmul_rn((float)((u[i].x - mean) * inv), g.x), bb.x);  // kernels.py:35
      o.y = fadd_rn(fmul_rn((float)((u[i].y - mean) * inv), g.y), bb.y);
      o.z = fadd_rn(fmul_rn((float)((u[i].z - mean) * inv), g.z), bb.z);
      o.w = fadd_rn(fmul_rn((float)((u[i].w - mean) * inv), g.w), bb.w);
      if (out) *reinterpret_cast<float4*>(out + row * ldo + c) = o;
      if (out16) {
        store_half4(out16, out16lo, row * ldo16 + c, o);
      }
    }
  }
}

// 128 threads per row, V float4 per thread (d = 512 * V): 4x the warps of the
// warp-per-row kernel for the decoder's few hundred rows (latency-bound op).
template <bool kBiasRes, int V>
__global__ void __launch_bounds__(128) layer_norm_row128_kernel(
    const float* __restrict__ x, int64_t ldx, const float* __restrict__ bias,
    const float* __restrict__ res, int64_t ldr, const float* __restrict__ gamma,
    const float* __restrict__ beta, double eps, int d, float* __restrict__ out, int64_t ldo,
    h16* __restrict__ out16, h16* __restrict__ out16lo, int64_t ldo16) {
  pdl_enter();
  __shared__ double red[2][4];
  const int64_t row = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 u[V];
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = (i * 128 + threadIdx.x) * 4;
    float4 a = *reinterpret_cast<const float4*>(x + row * ldx + c);
    if (kBiasRes) {
      const float4 b = *reinterpret_cast<const float4*>(bias + c);
      const float4 r = *reinterpret_cast<const float4*>(res + row * ldr + c);
      a.x = fadd_rn(fadd_rn(a.x, b.x), r.x);
      a.y = fadd_rn(fadd_rn(a.y, b.y), r.y);
      a.z = fadd_rn(fadd_rn(a.z, b.z), r.z);
      a.w = fadd_rn(fadd_rn(a.w, b.w), r.w);
    }
    u[i] = a;
    s += ((double)a.x + (double)a.y) + ((double)a.z + (double)a.w);
  }
  s = warp_sum(s);
  if (lane == 0) red[0][w] = s;
  __syncthreads();
  const double mean = ((red[0][0] + red[0][1]) + (red[0][2] + red[0][3])) / d;
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    double t0 = u[i].x - mean, t1 = u[i].y - mean, t2 = u[i].z - mean, t3 = u[i].w - mean;
    v += (t0 * t0 + t1 * t1) + (t2 * t2 + t3 * t3);
  }
  v = warp_sum(v);
  if (lane == 0) red[1][w] = v;
  __syncthreads();
  const double inv = 1.0 / sqrt(((red[1][0] + red[1][1]) + (red[1][2] + red[1][3])) / d + eps);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = (i * 128 + threadIdx.x) * 4;
    const float4 g = *reinterpret_cast<const float4*>(gamma + c);
    const float4 bb = *reinterpret_cast<const float4*>(beta + c);
    float4 o;
    o.x = fadd_rn(fmul_rn((float)((u[i].x - mean) * inv), g.x), bb.x);  // kernels.py:35
    o.y = fadd_rn(fmul_rn((float)((u[i].y - mean) * inv), g.y), bb.y);
    o.z = fadd_rn(fmul_rn((float)((u[i].z - mean) * inv), g.z), bb.z);
    o.w = fadd_rn(fmul_rn((float)((u[i].w - mean) * inv), g.w), bb.w);
    if (out) *reinterpret_cast<float4*>(out + row * ldo + c) = o;
    if (out16) {
      store_half4(out16, out16lo, row * ldo16 + c, o);
    }
  }
}

// Split-K consumer: x = the S fp32 partial slabs of a split-K GEMM ([S][rows][ld],
// slab s = K slice s), summed in split order, + bias, + residual, then the LN
// of layer_norm_row128_kernel — the same additions in the same order as the
// split-K kernel's DSMEM epilogue followed by fq_layer_norm.
template <int V, int NS>
__global__ void __launch_bounds__(128) layer_norm_slabs_row128_kernel(
    const float* __restrict__ x, int64_t ld, int64_t slab, const float* __restrict__ bias,
    const float* __restrict__ res, int64_t ldr, const float* __restrict__ gamma,
    const float* __restrict__ beta, double eps, int d, float* __restrict__ out, int64_t ldo,
    h16* __restrict__ out16, h16* __restrict__ out16lo, int64_t ldo16) {
  pdl_launch_dependents();
  __shared__ double red[2][4];
  const int64_t row = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // the (constant) bias / gamma / beta before the grid-dependency wait: their
  // fetch overlaps the producing GEMM's tail instead of adding a round trip
  float4 bv[V], gv[V], ev[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = (i * 128 + threadIdx.x) * 4;
    bv[i] = *reinterpret_cast<const float4*>(bias + c);
    gv[i] = *reinterpret_cast<const float4*>(gamma + c);
    ev[i] = *reinterpret_cast<const float4*>(beta + c);
  }
  pdl_wait();
  float4 u[V];
  double s = 0.0;
  float4 p[V][NS], rv[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = (i * 128 + threadIdx.x) * 4;
#pragma unroll
    for (int k = 0; k < NS; ++k) p[i][k] = __ldcg(reinterpret_cast<const float4*>(x + k * slab + row * ld + c));
    rv[i] = *reinterpret_cast<const float4*>(res + row * ldr + c);
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = (i * 128 + threadIdx.x) * 4;
    float4 a = p[i][0];
#pragma unroll
    for (int k = 1; k < NS; ++k) {
      a.x = fadd_rn(a.x, p[i][k].x);
      a.y = fadd_rn(a.y, p[i][k].y);
      a.z = fadd_rn(a.z, p[i][k].z);
      a.w = fadd_rn(a.w, p[i][k].w);
    }
    const float4 b = bv[i];
    const float4 r = rv[i];
    a.x = fadd_rn(fadd_rn(a.x, b.x), r.x);
    a.y = fadd_rn(fadd_rn(a.y, b.y), r.y);
    a.z = fadd_rn(fadd_rn(a.z, b.z), r.z);
    a.w = fadd_rn(fadd_rn(a.w, b.w), r.w);
    u[i] = a;
    s += ((double)a.x + (double)a.y) + ((double)a.z + (double)a.w);
  }
  s = warp_sum(s);
  if (lane == 0) red[0][w] = s;
  __syncthreads();
  const double mean = ((red[0][0] + red[0][1]) + (red[0][2] + red[0][3])) / d;
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    double t0 = u[i].x - mean, t1 = u[i].y - mean, t2 = u[i].z - mean, t3 = u[i].w - mean;
    v += (t0 * t0 + t1 * t1) + (t2 * t2 + t3 * t3);
  }
  v = warp_sum(v);
  if (lane == 0) red[1][w] = v;
  __syncthreads();
  const double inv = 1.0 / sqrt(((red[1][0] + red[1][1]) + (red[1][2] + red[1][3])) / d + eps);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = (i * 128 + threadIdx.x) * 4;
    const float4 g = gv[i];
    const float4 bb = ev[i];
    float4 o;
    o.x = fadd_rn(fmul_rn((float)((u[i].x - mean) * inv), g.x), bb.x);  // kernels.py:35
    o.y = fadd_rn(fmul_rn((float)((u[i].y - mean) * inv), g.y), bb.y);
    o.z = fadd_rn(fmul_rn((float)((u[i].z - mean) * inv), g.z), bb.z);
    o.w = fadd_rn(fmul_rn((float)((u[i].w - mean) * inv), g.w), bb.w);
    if (out) *reinterpret_cast<float4*>(out + row * ldo + c) = o;
    if (out16) {
      store_half4(out16, out16lo, row * ldo16 + c, o);
    }
  }
}

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <bool kBiasRes>
static void launch_ln(const float* x, int64_t ldx, const float* bias, const float* res,
                      int64_t ldr, const float* gamma, const float* beta, double eps,
                      int64_t rows, int64_t d, float* out, int64_t ldo, h16* out16,
                      int64_t ldo16, cudaStream_t s, h16* out16lo = nullptr) {
  bool align_ok = ldx % 4 == 0 && aligned16(x) && aligned16(gamma) && aligned16(beta) &&
                  (!out || (ldo % 4 == 0 && aligned16(out))) &&
                  (!out16 || (ldo16 % 4 == 0 && (reinterpret_cast<uintptr_t>(out16) & 7) == 0)) &&
                  (!out16lo || (reinterpret_cast<uintptr_t>(out16lo) & 7) == 0);
  if (kBiasRes) align_ok = align_ok && ldr % 4 == 0 && aligned16(res) && aligned16(bias);
  const bool warp_ok = align_ok && d % 128 == 0 && d <= 128 * kMaxV;
  const bool row128 = align_ok && (d == 512 || d == 1024 || d == 2048) &&
                      (rows < 4 * 148 * 8 || d == 2048);
  if (row128) {
    // few rows (decoder): 128 threads per row keep enough loads in flight
#define FQ_LN128(V)                                                                       \
  launch_kernel(layer_norm_row128_kernel<kBiasRes, V>, (unsigned)rows, 128, 0, s, 1u,                    \
      x, ldx, bias, res, ldr, gamma, beta, eps, (int)d, out, ldo, out16, out16lo, ldo16)
    if (d == 512) FQ_LN128(1);
    else if (d == 1024) FQ_LN128(2);
    else FQ_LN128(4);
#undef FQ_LN128
  } else if (warp_ok) {
    const int64_t threads = rows * 32;
    launch_kernel(layer_norm_warp_kernel<kBiasRes>, (unsigned)((threads + 255) / 256), 256, 0, s, 1u, 
        x, ldx, bias, res, ldr, gamma, beta, eps, rows, (int)d, out, ldo, out16, out16lo, ldo16);
  } else {
    int threads = d >= 1024 ? 256 : 128;
    launch_kernel(layer_norm_kernel<kBiasRes>, (unsigned)rows, threads, d * sizeof(float), s, 1u, 
        x, ldx, bias, res, ldr, gamma, beta, eps, (int)d, out, ldo, out16, out16lo, ldo16);
  }
}

// act(x + bias) (+ residual), kernels.py:39-53.
__global__ void bias_residual_act_kernel(const float* __restrict__ x, int64_t ldx,
                                         const float* __restrict__ bias,
                                         const float* __restrict__ res, int64_t ldr, int act,
                                         int64_t rows, int d, float* out, int64_t ldo) {
  pdl_enter();
  const int64_t n = rows * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / d;
    int j = (int)(i - r * d);
    float t = apply_act(fadd_rn(x[r * ldx + j], bias[j]), act);
    if (res) t = fadd_rn(t, res[r * ldr + j]);  // f64 sum of two fp32, rounded = RN fp32 add
    out[r * ldo + j] = t;
  }
}

// [batch*seq, parts*d] + bias -> parts x [batch, heads, seq, hd] (kernels.py:77-102).
__global__ void bias_reshape_kernel(const float* __restrict__ x, int64_t ldx,
                                    const float* __restrict__ bias, int64_t seq, int heads,
                                    int hd, int parts, int64_t n_rows, float* __restrict__ o0,
                                    float* __restrict__ o1, float* __restrict__ o2) {
  pdl_enter();
  const int d = heads * hd;
  const int64_t per_part = n_rows * d;
  const int64_t total = per_part * parts;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int part = (int)(idx / per_part);
    int64_t rem = idx - part * per_part;
    int64_t i = rem / d;  // input row (b*seq + s)
    int j = (int)(rem - i * d);
    float v = fadd_rn(x[i * ldx + part * d + j], bias[part * d + j]);
    int64_t b = i / seq, s = i - b * seq;
    int h = j / hd, e = j - h * hd;
    float* o = part == 0 ? o0 : (part == 1 ? o1 : o2);
    o[((b * heads + h) * seq + s) * hd + e] = v;
  }
}

// softmax(scores*scale + mask) per row, kernels.py:106-139: one warp per row.
__global__ void scale_mask_softmax_kernel(const float* __restrict__ sc, int64_t ld, float* out,
                                          int64_t ldo, int64_t rows, int64_t rows_per_b,
                                          int l, float scale, const float* __restrict__ mask,
                                          int* d_bad) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= rows) return;
  const float* s = sc + row * ld;
  const float* mk = mask ? mask + (row / rows_per_b) * l : nullptr;
  float m = -INFINITY;
  for (int j = lane; j < l; j += 32) {
    float t = fmul_rn(s[j], scale);
    if (mk) t = fadd_rn(t, mk[j]);
    m = fmaxf(m, t);
  }
  m = warp_max(m);
  if (m == -INFINITY) {  // kernels.py:121-123: counted, row left untouched
    if (lane == 0 && d_bad) atomicAdd(d_bad, 1);
    return;
  }
  double acc = 0.0;
  for (int j = lane; j < l; j += 32) {
    float t = fmul_rn(s[j], scale);
    if (mk) t = fadd_rn(t, mk[j]);
    acc += exp((double)t - (double)m);
  }
  const double inv = 1.0 / warp_sum(acc);
  float* o = out + row * ldo;
  for (int j = lane; j < l; j += 32) {
    float t = fmul_rn(s[j], scale);
    if (mk) t = fadd_rn(t, mk[j]);
    o[j] = (t == -INFINITY) ? 0.0f : (float)(exp((double)t - (double)m) * inv);
  }
}

// out[i] = emb[tok[i]] * scale + pos[i % seq + off], kernels.py:143-151.
__global__ void embed_kernel(const int64_t* __restrict__ tok, int64_t n,
                             const float* __restrict__ emb, int d, float scale,
                             const float* __restrict__ pos, int64_t off,
                             const int32_t* __restrict__ d_off, int64_t seq, float* out,
                             h16* out16) {
  pdl_enter();
  const int64_t base = d_off ? (int64_t)(*d_off) : off;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * d;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx / d;
    int j = (int)(idx - i * d);
    int64_t p = i % seq + base;
    float v = fadd_rn(fmul_rn(emb[tok[i] * d + j], scale), pos[p * d + j]);
    if (out) out[idx] = v;
    if (out16) out16[idx] = f2h(v);
  }
}

// KV cache refresh, kernels.py:189-211: dst [R, h, S, hd].
__global__ void kv_kernel(const float* __restrict__ sk, const float* __restrict__ sv,
                          const float* __restrict__ nk, const float* __restrict__ nv,
                          const int64_t* __restrict__ parents, int64_t cur, int64_t rows,
                          int heads, int64_t S, int hd, float* dk, float* dv) {
  pdl_enter();
  const int64_t hist = parents ? cur + 1 : 1;  // positions written per (r, h)
  const int64_t total = rows * heads * hist * hd;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int e = (int)(idx % hd);
    int64_t t = (idx / hd) % hist;
    int64_t rh = idx / (hd * hist);
    int h = (int)(rh % heads);
    int64_t r = rh / heads;
    int64_t pos = parents ? t : cur;
    int64_t dst = ((r * heads + h) * S + pos) * hd + e;
    if (pos == cur) {
      int64_t src = (r * heads + h) * hd + e;  // new [R, h, 1, hd]
      dk[dst] = nk[src];
      dv[dst] = nv[src];
    } else {
      int64_t src = ((parents[r] * heads + h) * S + pos) * hd + e;
      dk[dst] = sk[src];
      dv[dst] = sv[src];
    }
  }
}

// Diversity penalty (kernels.py:215-219): out = logits - f32(lam) * count[j],
// numba-typed as f32 * i32 -> f64, f32 - f64 -> f64, stored as f32.
__global__ void penalize_counts_kernel(const float* __restrict__ logits, int64_t ld, int64_t rows,
                                       int64_t vocab, const int32_t* __restrict__ counts,
                                       float lam, float* __restrict__ out, int64_t ldo) {
  pdl_enter();
  const int64_t n = rows * vocab;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / vocab, j = i - r * vocab;
    out[r * ldo + j] = (float)((double)logits[r * ld + j] - (double)lam * (double)counts[j]);
  }
}

static inline int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = 148LL * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_layer_norm(const float* x, int64_t ldx, const float* gamma, const float* beta,
                  double eps, int64_t rows, int64_t d, float* out, int64_t ldo, void* out16,
                  int64_t ldo16, fq_stream_t stream) {
  FQ_CHECK_ARG(x && gamma && beta && rows >= 0 && d > 0 && d <= 12288 && (out || out16),
               FQ_ERR_DIMENSION, "fq_layer_norm: bad shape rows=%lld d=%lld", (long long)rows,
               (long long)d);
  FQ_CHECK_ARG(eps >= 0, FQ_ERR_DIMENSION, "eps must be non-negative");
  if (rows == 0) return FQ_OK;
  launch_ln<false>(x, ldx, nullptr, nullptr, 0, gamma, beta, eps, rows, d, out, ldo,
                   reinterpret_cast<fq::h16*>(out16), ldo16, as_stream(stream));
  return launch_status("fq_layer_norm");
}

int fq_bias_residual_layer_norm(const float* x, int64_t ldx, const float* bias,
                                const float* residual, int64_t ldr, const float* gamma,
                                const float* beta, double eps, int64_t rows, int64_t d,
                                float* out, int64_t ldo, void* out16, int64_t ldo16,
                                fq_stream_t stream) {
  FQ_CHECK_ARG(x && bias && residual && gamma && beta && d > 0 && d <= 12288 && (out || out16),
               FQ_ERR_DIMENSION, "fq_bias_residual_layer_norm: bad args");
  if (rows == 0) return FQ_OK;
  launch_ln<true>(x, ldx, bias, residual, ldr, gamma, beta, eps, rows, d, out, ldo,
                  reinterpret_cast<fq::h16*>(out16), ldo16, as_stream(stream));
  return launch_status("fq_bias_residual_layer_norm");
}

static int splitk_ln(const float* slabs, int nslab, int64_t ld, const float* bias,
                     const float* residual, int64_t ldr, const float* gamma, const float* beta,
                     double eps, int64_t rows, int64_t d, float* out, int64_t ldo, void* out16,
                     void* out16lo, int64_t ldo16, fq_stream_t stream) {
  FQ_CHECK_ARG(slabs && bias && residual && gamma && beta && rows >= 0 && (out || out16) &&
                   (nslab == 2 || nslab == 4) && (d == 512 || d == 1024 || d == 2048) &&
                   ld >= d && ld % 4 == 0 && ldr % 4 == 0 && aligned16(slabs) &&
                   aligned16(bias) && aligned16(residual) && aligned16(gamma) &&
                   aligned16(beta) && (!out || (ldo % 4 == 0 && aligned16(out))) &&
                   (!out16 || (ldo16 % 4 == 0 && (reinterpret_cast<uintptr_t>(out16) & 7) == 0)) &&
                   (!out16lo || (out16 && (reinterpret_cast<uintptr_t>(out16lo) & 7) == 0)),
               FQ_ERR_DIMENSION, "fq_splitk_bias_residual_layer_norm: bad args");
  FQ_CHECK_ARG(eps >= 0, FQ_ERR_DIMENSION, "eps must be non-negative");
  if (rows == 0) return FQ_OK;
  auto* o16 = reinterpret_cast<fq::h16*>(out16);
  auto* o16lo = reinterpret_cast<fq::h16*>(out16lo);
  const int64_t slab = rows * ld;
  cudaStream_t s = as_stream(stream);
#define FQ_LNS(V, NS)                                                                         \
  launch_kernel(layer_norm_slabs_row128_kernel<V, NS>, (unsigned)rows, 128, 0, s, 1u, slabs, ld, \
                slab, bias, residual, ldr, gamma, beta, eps, (int)d, out, ldo, o16, o16lo, ldo16)
  if (nslab == 4) {
    if (d == 512) FQ_LNS(1, 4);
    else if (d == 1024) FQ_LNS(2, 4);
    else FQ_LNS(4, 4);
  } else {
    if (d == 512) FQ_LNS(1, 2);
    else if (d == 1024) FQ_LNS(2, 2);
    else FQ_LNS(4, 2);
  }
#undef FQ_LNS
  return launch_status("fq_splitk_bias_residual_layer_norm");
}

int fq_splitk_bias_residual_layer_norm(const float* slabs, int nslab, int64_t ld,
                                       const float* bias, const float* residual, int64_t ldr,
                                       const float* gamma, const float* beta, double eps,
                                       int64_t rows, int64_t d, float* out, int64_t ldo,
                                       void* out16, int64_t ldo16, fq_stream_t stream) {
  return splitk_ln(slabs, nslab, ld, bias, residual, ldr, gamma, beta, eps, rows, d, out, ldo,
                   out16, nullptr, ldo16, stream);
}

int fq_splitk_bias_residual_layer_norm_xh(const float* slabs, int nslab, int64_t ld,
                                          const float* bias, const float* residual, int64_t ldr,
                                          const float* gamma, const float* beta, double eps,
                                          int64_t rows, int64_t d, float* out, int64_t ldo,
                                          void* out16, void* out16_lo, int64_t ldo16,
                                          fq_stream_t stream) {
  return splitk_ln(slabs, nslab, ld, bias, residual, ldr, gamma, beta, eps, rows, d, out, ldo,
                   out16, out16_lo, ldo16, stream);
}

int fq_layer_norm_xh(const float* x, int64_t ldx, const float* gamma, const float* beta,
                     double eps, int64_t rows, int64_t d, float* out, int64_t ldo, void* out16,
                     void* out16_lo, int64_t ldo16, fq_stream_t stream) {
  FQ_CHECK_ARG(x && gamma && beta && rows >= 0 && d > 0 && d <= 12288 && (out || out16) &&
                   (!out16_lo || out16),
               FQ_ERR_DIMENSION, "fq_layer_norm_xh: bad args");
  if (rows == 0) return FQ_OK;
  launch_ln<false>(x, ldx, nullptr, nullptr, 0, gamma, beta, eps, rows, d, out, ldo,
                   reinterpret_cast<fq::h16*>(out16), ldo16, as_stream(stream),
                   reinterpret_cast<fq::h16*>(out16_lo));
  return launch_status("fq_layer_norm_xh");
}

int fq_bias_residual_act(const float* x, int64_t ldx, const float* bias, const float* residual,
                         int64_t ldr, int act, int64_t rows, int64_t d, float* out, int64_t ldo,
                         fq_stream_t stream) {
  FQ_CHECK_ARG(x && bias && out && d > 0, FQ_ERR_DIMENSION, "fq_bias_residual_act: bad args");
  FQ_CHECK_ARG(act >= 0 && act <= 2, FQ_ERR_PARAMETER, "unknown activation %d", act);
  if (rows == 0) return FQ_OK;
  launch_kernel(bias_residual_act_kernel, grid_for(rows * d, 256), 256, 0, as_stream(stream), 1u, 
      x, ldx, bias, residual, ldr, act, rows, (int)d, out, ldo);
  return launch_status("fq_bias_residual_act");
}

int fq_qkv_bias_reshape(const float* qkv, int64_t ldq, const float* bias, int64_t batch,
                        int64_t seq, int64_t heads, int64_t head_dim, float* q, float* k,
                        float* v, fq_stream_t stream) {
  FQ_CHECK_ARG(qkv && bias && q && k && v && batch > 0 && seq > 0 && heads > 0 && head_dim > 0,
               FQ_ERR_DIMENSION, "fq_qkv_bias_reshape: bad args");
  int64_t n = batch * seq * heads * head_dim * 3;
  launch_kernel(bias_reshape_kernel, grid_for(n, 256), 256, 0, as_stream(stream), 1u, 
      qkv, ldq, bias, seq, (int)heads, (int)head_dim, 3, batch * seq, q, k, v);
  return launch_status("fq_qkv_bias_reshape");
}

int fq_bias_reshape_heads(const float* x, int64_t ldx, const float* bias, int64_t batch,
                          int64_t seq, int64_t heads, int64_t head_dim, float* out,
                          fq_stream_t stream) {
  FQ_CHECK_ARG(x && bias && out && batch > 0 && seq > 0 && heads > 0 && head_dim > 0,
               FQ_ERR_DIMENSION, "fq_bias_reshape_heads: bad args");
  int64_t n = batch * seq * heads * head_dim;
  launch_kernel(bias_reshape_kernel, grid_for(n, 256), 256, 0, as_stream(stream), 1u, 
      x, ldx, bias, seq, (int)heads, (int)head_dim, 1, batch * seq, out, nullptr, nullptr);
  return launch_status("fq_bias_reshape_heads");
}

int fq_scale_mask_softmax(const float* scores, int64_t ld, float* out, int64_t ldo, int64_t b,
                          int64_t h, int64_t q, int64_t l, float scale, const float* mask,
                          int* d_bad, fq_stream_t stream) {
  FQ_CHECK_ARG(scores && out && b > 0 && h > 0 && q > 0 && l > 0 && ld >= l && ldo >= l,
               FQ_ERR_DIMENSION, "fq_scale_mask_softmax: bad shape");
  int64_t rows = b * h * q;
  int64_t threads = rows * 32;
  launch_kernel(scale_mask_softmax_kernel, (unsigned)((threads + 255) / 256), 256, 0, as_stream(stream), 1u, 
      scores, ld, out, ldo, rows, h * q, (int)l, scale, mask, d_bad);
  return launch_status("fq_scale_mask_softmax");
}

int fq_embed_scale_pos(const int64_t* tokens, int64_t n, const float* emb, int64_t d,
                       float scale, const float* pos, int64_t pos_offset, const int32_t* d_off,
                       int64_t seq, float* out, void* out16, fq_stream_t stream) {
  FQ_CHECK_ARG(tokens && emb && pos && d > 0 && seq > 0 && (out || out16), FQ_ERR_DIMENSION,
               "fq_embed_scale_pos: bad args");
  if (n == 0) return FQ_OK;
  launch_kernel(embed_kernel, grid_for(n * d, 256), 256, 0, as_stream(stream), 1u, 
      tokens, n, emb, (int)d, scale, pos, pos_offset, d_off, seq, out,
      reinterpret_cast<fq::h16*>(out16));
  return launch_status("fq_embed_scale_pos");
}

int fq_penalize_counts(const float* logits, int64_t ld, int64_t rows, int64_t vocab,
                       const int32_t* counts, float lam, float* out, int64_t ldo,
                       fq_stream_t stream) {
  FQ_CHECK_ARG(logits && counts && out && rows >= 0 && vocab >= 1 && ld >= vocab && ldo >= vocab,
               FQ_ERR_DIMENSION, "fq_penalize_counts: bad args");
  if (rows == 0) return FQ_OK;
  launch_kernel(penalize_counts_kernel, grid_for(rows * vocab, 256), 256, 0, as_stream(stream),
                1u, logits, ld, rows, vocab, counts, lam, out, ldo);
  return launch_status("fq_penalize_counts");
}

int fq_kv_append(const float* new_k, const float* new_v, int64_t cur, int64_t rows,
                 int64_t heads, int64_t max_seq, int64_t head_dim, float* dst_k, float* dst_v,
                 fq_stream_t stream) {
  FQ_CHECK_ARG(cur >= 0 && cur < max_seq, FQ_ERR_CAPACITY, "KV cache full at %lld positions",
               (long long)cur);
  int64_t n = rows * heads * head_dim;
  launch_kernel(kv_kernel, grid_for(n, 256), 256, 0, as_stream(stream), 1u, 
      nullptr, nullptr, new_k, new_v, nullptr, cur, rows, (int)heads, max_seq, (int)head_dim,
      dst_k, dst_v);
  return launch_status("fq_kv_append");
}

int fq_kv_gather_append(const float* src_k, const float* src_v, const float* new_k,
                        const float* new_v, const int64_t* parents, int64_t cur, int64_t rows,
                        int64_t heads, int64_t max_seq, int64_t head_dim, float* dst_k,
                        float* dst_v, fq_stream_t stream) {
  FQ_CHECK_ARG(cur >= 0 && cur < max_seq, FQ_ERR_CAPACITY, "KV cache full at %lld positions",
               (long long)cur);
  FQ_CHECK_ARG(src_k != dst_k && src_v != dst_v, FQ_ERR_ALIASING,
               "ping-pong gather must not read and write the same slot");
  int64_t n = rows * heads * (cur + 1) * head_dim;
  launch_kernel(kv_kernel, grid_for(n, 256), 256, 0, as_stream(stream), 1u, 
      src_k, src_v, new_k, new_v, parents, cur, rows, (int)heads, max_seq, (int)head_dim, dst_k,
      dst_v);
  return launch_status("fq_kv_gather_append");
}

}  // extern "C"
