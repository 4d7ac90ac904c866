// Fused attention for the device engine.
//
// The reference runs attention as gemm_batched(QK^T) -> scale_mask_softmax ->
// gemm_batched(P.V) writing a merged-head strided view (model.py:329-336,
// :572-580, :597-604). These kernels do the same three steps in one pass per
// (item, head) so the [b, h, q, l] score tensor never reaches HBM; the softmax
// keeps the kernels.py:106-139 numerics in exact mode (fp32 scale+mask, f64
// exp and sum, F32(exp * (1/sum)), masked -> 0). Every dot product is an fp32
// FMA chain over the head dimension in order; the P.V sum runs over keys in
// ascending order.
//
// Decoder self-attention replaces the reference's ping-pong KV gather
// (kernels.py:189-201: ~50 GB/request at C2) with a copy-free
// history table: slot (t, r) of the cache is written once, by row r at step t,
// and hist[r, t] names the physical row whose slot holds row r's position t.
// Beam reorder then moves B*K*max_len int32 instead of the K/V history.
//
// All three kernels are bandwidth/latency bound: head slices are staged with
// 128-bit loads (8 fp16 or 4 fp32 per load), all issued before first use.
#include <cuda.h>
#include <stdlib.h>

#include "fq_common.cuh"

namespace fq {

template <typename T>
__device__ __forceinline__ float ld_as_f32(const T* p);
template <>
__device__ __forceinline__ float ld_as_f32<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_as_f32<h16>(const h16* p) {
  return h2f(*p);
}

// 16 bytes -> EV floats
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& raw, float* o);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& raw, float* o) {
  o[0] = __uint_as_float(raw.x); o[1] = __uint_as_float(raw.y);
  o[2] = __uint_as_float(raw.z); o[3] = __uint_as_float(raw.w);
}
template <>
__device__ __forceinline__ void unpack16<h16>(const uint4& raw, float* o) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(*reinterpret_cast<const h16x2*>(&w[i]));
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}

// Stage a [rows, hd] slice (row stride ld elements) into fp32 smem [rows][hp].
template <typename T>
__device__ __forceinline__ void load_slice(const T* __restrict__ src, int64_t ld, int rows,
                                           int hd, float* dst, int hp) {
  constexpr int EV = 16 / sizeof(T);
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)(ld * sizeof(T))) & 15) == 0 &&
                   hd % EV == 0;
  if (vec) {
    const int vpr = hd / EV;
    const int n = rows * vpr;
    constexpr int U = 4;
    for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
      uint4 raw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < n) raw[u] = *reinterpret_cast<const uint4*>(src + (int64_t)(i / vpr) * ld + (i % vpr) * EV);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < n) {
          float f[EV];
          unpack16<T>(raw[u], f);
          float* d = dst + (i / vpr) * hp + (i % vpr) * EV;
#pragma unroll
          for (int j = 0; j < EV; ++j) d[j] = f[j];
        }
      }
    }
  } else {
    for (int i = threadIdx.x; i < rows * hd; i += blockDim.x)
      dst[(i / hd) * hp + i % hd] = ld_as_f32(src + (int64_t)(i / hd) * ld + i % hd);
  }
}

// Softmax over `n` scores held in smem `s` (one warp). Writes probabilities
// in place. Returns false when every score is -inf (fully masked row).
__device__ __forceinline__ bool warp_softmax(float* s, int n, bool exact) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY;
  for (int j = lane; j < n; j += 32) m = fmaxf(m, s[j]);
  m = warp_max(m);
  if (m == -INFINITY) return false;
  if (exact) {
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc += exp((double)s[j] - (double)m);
    const double inv = 1.0 / warp_sum(acc);
    __syncwarp();
    for (int j = lane; j < n; j += 32) {
      float t = s[j];
      s[j] = (t == -INFINITY) ? 0.0f : (float)(exp((double)t - (double)m) * inv);
    }
  } else {
    float acc = 0.0f;
    for (int j = lane; j < n; j += 32) acc += __expf(s[j] - m);
    const float inv = 1.0f / warp_sum(acc);
    __syncwarp();
    for (int j = lane; j < n; j += 32) {
      float t = s[j];
      s[j] = (t == -INFINITY) ? 0.0f : __expf(t - m) * inv;
    }
  }
  __syncwarp();
  return true;
}

// One warp: rows `Qs` of queries against staged K/V of one head; used by the
// encoder (queries = the item's positions) and cross attention (queries = beams).
__device__ __forceinline__ void attend_rows(const float* Qs, const float* Ks, const float* Vs,
                                            float* Ss, int seq, int hd, int hp, float scale,
                                            const float* mk, bool exact, float* out,
                                            h16* out16, int* d_bad) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < seq; j += 32) {
    float acc = 0.0f;
    for (int e = 0; e < hd; ++e) acc = fmaf(Qs[e], Ks[j * hp + e], acc);
    float t = fmul_rn(acc, scale);
    if (mk) t = fadd_rn(t, mk[j]);
    Ss[j] = t;
  }
  __syncwarp();
  if (!warp_softmax(Ss, seq, exact)) {
    if (lane == 0 && d_bad) atomicAdd(d_bad, 1);
    return;
  }
  for (int e = lane; e < hd; e += 32) {
    float acc = 0.0f;
    for (int j = 0; j < seq; ++j) acc = fmaf(Ss[j], Vs[j * hp + e], acc);
    if (out) out[e] = acc;
    if (out16) out16[e] = f2h(acc);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Encoder self-attention: CTA per (item, head); K/V of the head in smem.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) encoder_attention_kernel(
    const float* __restrict__ qkv, int64_t ldq, int seq, int heads, int hd, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int exact, int* d_bad) {
  pdl_enter();
  extern __shared__ float sm[];
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int d = heads * hd;
  const int hp = hd + 1;  // padded row: conflict-free column walks
  float* Ks = sm;
  float* Vs = Ks + seq * hp;
  float* Qa = Vs + seq * hp;  // all queries of the head, [seq][hd]
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
  float* Ss = Qa + seq * hd + w * seq;
  const float* base = qkv + (int64_t)b * seq * ldq;
  load_slice<float>(base + d + h * hd, ldq, seq, hd, Ks, hp);
  load_slice<float>(base + 2 * d + h * hd, ldq, seq, hd, Vs, hp);
  load_slice<float>(base + h * hd, ldq, seq, hd, Qa, hd);
  __syncthreads();
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  for (int i = w; i < seq; i += nw) {
    const int64_t orow = ((int64_t)b * seq + i) * ldo + h * hd;
    attend_rows(Qa + i * hd, Ks, Vs, Ss, seq, hd, hp, scale, mk, exact,
                out ? out + orow : nullptr, out16 ? out16 + orow : nullptr, d_bad);
  }
}

// ---------------------------------------------------------------------------
// Decoder self-attention. Lane-parallel over cache positions: lane t computes
// the full fp32 dot q.k_t (keys gathered through hist with 128-bit loads), the
// warp softmaxes, then P.V walks positions in order with coalesced V rows.
// 4 consecutive rows (one item at beam 4) per CTA so beams that share physical
// slots hit in L1.
// ---------------------------------------------------------------------------
template <typename KV, int HD>
__global__ void __launch_bounds__(128) decoder_self_attention_fast(
    const float* __restrict__ sqkv, int64_t ldq, KV* __restrict__ kc, KV* __restrict__ vc,
    const int32_t* __restrict__ hist, const int32_t* __restrict__ d_cur, int rows, int heads,
    int max_len, float scale, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int exact) {
  pdl_enter();
  extern __shared__ float sm[];
  constexpr int EV = 16 / sizeof(KV);  // elements per 128-bit load
  constexpr int EPL = (HD + 31) / 32;  // output elements per lane in P.V
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + w;
  const int h = blockIdx.y;
  if (r >= rows) return;
  const int cur = *d_cur;
  const int d = heads * HD;
  float* Ss = sm + w * (2 * max_len + 2);
  int* Ps = reinterpret_cast<int*>(Ss + max_len + 1);
  const float* rowp = sqkv + (int64_t)r * ldq + h * HD;
  // q (all lanes hold the full vector; L1 broadcast)
  float q[HD];
#pragma unroll
  for (int e = 0; e < HD; e += 4) {
    const float4 v = *reinterpret_cast<const float4*>(rowp + e);
    q[e] = v.x; q[e + 1] = v.y; q[e + 2] = v.z; q[e + 3] = v.w;
  }
  // this step's K/V go to slot (cur, r)
  const int64_t slot_cur = ((int64_t)cur * rows + r) * d + h * HD;
  for (int e = lane; e < HD; e += 32) {
    if constexpr (sizeof(KV) == 4) {
      kc[slot_cur + e] = rowp[d + e];
      vc[slot_cur + e] = rowp[2 * d + e];
    } else {
      kc[slot_cur + e] = f2h(rowp[d + e]);
      vc[slot_cur + e] = f2h(rowp[2 * d + e]);
    }
  }
  const int32_t* hr = hist + (int64_t)r * max_len;
  // scores: lane t
  for (int t0 = 0; t0 <= cur; t0 += 32) {
    const int t = t0 + lane;
    if (t <= cur) {
      const int phys = t == cur ? r : hr[t];
      Ps[t] = phys;
      float acc = 0.0f;
      if (t == cur) {
#pragma unroll
        for (int e = 0; e < HD; ++e) {
          float kv = rowp[d + e];
          if constexpr (sizeof(KV) == 2) kv = h2f(f2h(kv));  // the stored (rounded) key
          acc = fmaf(q[e], kv, acc);
        }
      } else {
        const KV* kp = kc + ((int64_t)t * rows + phys) * d + h * HD;
        uint4 raw[HD / EV];
#pragma unroll
        for (int i = 0; i < HD / EV; ++i) raw[i] = *reinterpret_cast<const uint4*>(kp + i * EV);
#pragma unroll
        for (int i = 0; i < HD / EV; ++i) {
          float f[EV];
          unpack16<KV>(raw[i], f);
#pragma unroll
          for (int j = 0; j < EV; ++j) acc = fmaf(q[i * EV + j], f[j], acc);
        }
      }
      Ss[t] = fmul_rn(acc, scale);
    }
  }
  __syncwarp();
  warp_softmax(Ss, cur + 1, exact);  // no mask: causality is implicit (model.py:576)
  float acc[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) acc[i] = 0.0f;
#pragma unroll 4
  for (int t = 0; t <= cur; ++t) {
    const float p = Ss[t];
    const KV* vp = vc + ((int64_t)t * rows + Ps[t]) * d + h * HD;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = lane + 32 * i;
      if (e < HD) acc[i] = fmaf(p, ld_as_f32(vp + e), acc[i]);
    }
  }
  const int64_t o = (int64_t)r * ldo + h * HD;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const int e = lane + 32 * i;
    if (e < HD) {
      if (out) out[o + e] = acc[i];
      if (out16) out16[o + e] = f2h(acc[i]);
    }
  }
}

// ---------------------------------------------------------------------------
// Cross-attention: CTA per (item, head), warp per beam row; the item's K/V
// head slice is staged once in smem and shared by all beams.
// ---------------------------------------------------------------------------
template <typename KV>
__global__ void __launch_bounds__(256) cross_attention_kernel(
    const float* __restrict__ cq, int64_t ldcq, const KV* __restrict__ ck,
    const KV* __restrict__ cv, int64_t ldkv, int beam, int seq, int heads, int hd, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int exact, int* d_bad) {
  pdl_enter();
  extern __shared__ float sm[];
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int hp = hd + 1;
  float* Ks = sm;
  float* Vs = Ks + seq * hp;
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Ss = Vs + seq * hp + w * (seq + hd);
  float* Qs = Ss + seq;
  load_slice<KV>(ck + (int64_t)b * seq * ldkv + h * hd, ldkv, seq, hd, Ks, hp);
  load_slice<KV>(cv + (int64_t)b * seq * ldkv + h * hd, ldkv, seq, hd, Vs, hp);
  __syncthreads();
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  for (int i = w; i < beam; i += nw) {
    const int64_t r = (int64_t)b * beam + i;
    for (int e = lane; e < hd; e += 32) Qs[e] = cq[r * ldcq + h * hd + e];
    __syncwarp();
    attend_rows(Qs, Ks, Vs, Ss, seq, hd, hp, scale, mk, exact,
                out ? out + r * ldo + h * hd : nullptr, out16 ? out16 + r * ldo + h * hd : nullptr,
                d_bad);
  }
}

// Cross-attention, specialised: K/V staged raw (16-byte copies, K rows padded
// by 16 B so 128-bit row reads are conflict-free), each thread scores one key
// for two beams per pass (one K load feeds two FMA chains), one warp per beam
// softmax, and P.V with paired columns (f16x2 / float2 loads).
template <typename KV, int HD>
__global__ void __launch_bounds__(128) cross_attention_fast(
    const float* __restrict__ cq, int64_t ldcq, const KV* __restrict__ ck,
    const KV* __restrict__ cv, int64_t ldkv, int beam, int seq, int heads, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int exact, int* d_bad) {
  pdl_enter();
  constexpr int EV = 16 / sizeof(KV);
  constexpr int KP = HD + EV;  // padded K row (elements)
  extern __shared__ __align__(16) uint8_t smraw[];
  KV* Kt = reinterpret_cast<KV*>(smraw);
  KV* Vt = Kt + seq * KP;
  float* Qs = reinterpret_cast<float*>(Vt + seq * HD);
  float* Ps = Qs + beam * HD;
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // stage K/V (raw 16-byte copies, all issued before the first store)
  {
    constexpr int VPR = HD / EV;
    const int n = seq * VPR;
    const KV* kb = ck + (int64_t)b * seq * ldkv + h * HD;
    const KV* vb = cv + (int64_t)b * seq * ldkv + h * HD;
    for (int i0 = tid; i0 < n; i0 += 4 * 128) {
      uint4 rk[4], rv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 128;
        if (i < n) {
          const int r = i / VPR, c = (i % VPR) * EV;
          rk[u] = *reinterpret_cast<const uint4*>(kb + (int64_t)r * ldkv + c);
          rv[u] = *reinterpret_cast<const uint4*>(vb + (int64_t)r * ldkv + c);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 128;
        if (i < n) {
          const int r = i / VPR, c = (i % VPR) * EV;
          *reinterpret_cast<uint4*>(Kt + r * KP + c) = rk[u];
          *reinterpret_cast<uint4*>(Vt + r * HD + c) = rv[u];
        }
      }
    }
    for (int i = tid; i < beam * (HD / 4); i += 128) {
      const int bi = i / (HD / 4), c = (i % (HD / 4)) * 4;
      *reinterpret_cast<float4*>(Qs + bi * HD + c) =
          *reinterpret_cast<const float4*>(cq + ((int64_t)b * beam + bi) * ldcq + h * HD + c);
    }
  }
  __syncthreads();
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  // scores: thread -> (key j, beam pair)
  const int npairs = (beam + 1) / 2;
  for (int p = tid; p < seq * npairs; p += 128) {
    const int j = p % seq, b0 = 2 * (p / seq), b1 = b0 + 1;
    const bool two = b1 < beam;
    const float* q0 = Qs + b0 * HD;
    const float* q1 = Qs + (two ? b1 : b0) * HD;
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int e = 0; e < HD; e += EV) {
      float kf[EV];
      unpack16<KV>(*reinterpret_cast<const uint4*>(Kt + j * KP + e), kf);
#pragma unroll
      for (int t = 0; t < EV; ++t) {
        a0 = fmaf(q0[e + t], kf[t], a0);
        a1 = fmaf(q1[e + t], kf[t], a1);
      }
    }
    float t0 = fmul_rn(a0, scale), t1 = fmul_rn(a1, scale);
    if (mk) {
      t0 = fadd_rn(t0, mk[j]);
      t1 = fadd_rn(t1, mk[j]);
    }
    Ps[b0 * seq + j] = t0;
    if (two) Ps[b1 * seq + j] = t1;
  }
  __syncthreads();
  for (int bi = w; bi < beam; bi += 4) {
    if (!warp_softmax(Ps + bi * seq, seq, exact) && lane == 0 && d_bad) atomicAdd(d_bad, 1);
  }
  __syncthreads();
  // P.V: thread -> (beam, column pair)
  constexpr int TPB = HD / 2;  // threads per beam row
  for (int p = tid; p < beam * TPB; p += 128) {
    const int bi = p / TPB, e = (p % TPB) * 2;
    const float* pr = Ps + bi * seq;
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll 4
    for (int j = 0; j < seq; ++j) {
      const float pj = pr[j];
      float v0, v1;
      if constexpr (sizeof(KV) == 2) {
        const uint32_t raw = *reinterpret_cast<const uint32_t*>(Vt + j * HD + e);
        const float2 f = __half22float2(*reinterpret_cast<const h16x2*>(&raw));
        v0 = f.x;
        v1 = f.y;
      } else {
        const float2 f = *reinterpret_cast<const float2*>(Vt + j * HD + e);
        v0 = f.x;
        v1 = f.y;
      }
      a0 = fmaf(pj, v0, a0);
      a1 = fmaf(pj, v1, a1);
    }
    const int64_t o = ((int64_t)b * beam + bi) * ldo + h * HD + e;
    if (out) {
      out[o] = a0;
      out[o + 1] = a1;
    }
    if (out16) *reinterpret_cast<h16x2*>(out16 + o) = __floats2half2_rn(a0, a1);
  }
}

// Generic decoder self-attention (any head_dim <= 128), warp-reduced dots.
template <typename KV>
__global__ void __launch_bounds__(128) decoder_self_attention_kernel(
    const float* __restrict__ sqkv, int64_t ldq, KV* __restrict__ kc, KV* __restrict__ vc,
    const int32_t* __restrict__ hist, const int32_t* __restrict__ d_cur, int rows, int heads,
    int hd, int max_len, float scale, float* __restrict__ out,
    h16* __restrict__ out16, int64_t ldo, int exact) {
  pdl_enter();
  extern __shared__ float sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + w;
  const int h = blockIdx.y;
  if (r >= rows) return;
  const int cur = *d_cur;
  const int d = heads * hd;
  float* Ss = sm + w * (max_len + 1);
  const float* row = sqkv + (int64_t)r * ldq;
  const int64_t slot_cur = ((int64_t)cur * rows + r) * d + h * hd;
  constexpr int EPL = 4;
  float q[EPL], kn[EPL], vn[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    int e = lane + 32 * i;
    q[i] = kn[i] = vn[i] = 0.0f;
    if (e < hd) {
      q[i] = row[h * hd + e];
      kn[i] = row[d + h * hd + e];
      vn[i] = row[2 * d + h * hd + e];
      if constexpr (sizeof(KV) == 4) {
        kc[slot_cur + e] = kn[i];
        vc[slot_cur + e] = vn[i];
      } else {
        kc[slot_cur + e] = f2h(kn[i]);
        vc[slot_cur + e] = f2h(vn[i]);
        kn[i] = h2f(f2h(kn[i]));
        vn[i] = h2f(f2h(vn[i]));
      }
    }
  }
  const int32_t* hr = hist + (int64_t)r * max_len;
  for (int t = 0; t <= cur; ++t) {
    const KV* kp = kc + ((int64_t)t * rows + (t == cur ? r : hr[t])) * d + h * hd;
    float part = 0.0f;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      int e = lane + 32 * i;
      if (e < hd) part = fmaf(q[i], t == cur ? kn[i] : ld_as_f32(kp + e), part);
    }
    part = warp_sum(part);
    if (lane == 0) Ss[t] = fmul_rn(part, scale);
  }
  __syncwarp();
  warp_softmax(Ss, cur + 1, exact);
  float acc[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) acc[i] = 0.0f;
  for (int t = 0; t <= cur; ++t) {
    const float p = Ss[t];
    const KV* vp = vc + ((int64_t)t * rows + (t == cur ? r : hr[t])) * d + h * hd;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      int e = lane + 32 * i;
      if (e < hd) acc[i] = fmaf(p, t == cur ? vn[i] : ld_as_f32(vp + e), acc[i]);
    }
  }
  const int64_t o = (int64_t)r * ldo + h * hd;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    int e = lane + 32 * i;
    if (e < hd) {
      if (out) out[o + e] = acc[i];
      if (out16) out16[o + e] = f2h(acc[i]);
    }
  }
}

// ---------------------------------------------------------------------------
// Encoder self-attention, register-tiled: CTA per (item, head); Q/K/V head
// slices in smem; every thread owns a 4-row x NC-column block of the score
// tile (columns strided by 16 so the K reads are bank-conflict free) and a
// 4-row x HC-column block of the output. Same arithmetic as attend_rows —
// each score an fp32 FMA chain over e in order, each output an FMA chain over
// keys in order, softmax by warp_softmax — so both precision modes keep the
// exact-mode numerics; ~10x fewer shared-memory reads than one dot per lane.
// ---------------------------------------------------------------------------
template <int NC, int HC>
__global__ void __launch_bounds__(256, 4) encoder_attention_tiled(
    const float* __restrict__ qkv, int64_t ldq, int seq, int heads, int hd, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int exact, int* d_bad) {
  pdl_enter();
  extern __shared__ float sm[];
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int d = heads * hd;
  const int hp = hd + 1, sp = seq + 1;
  float* Qs = sm;               // [seq][hp]; reused as scores [seq][sp] (seq <= hd + ... checked)
  float* Ks = Qs + seq * (hp > sp ? hp : sp);
  float* Vs = Ks + seq * hp;
  int* bad_row = reinterpret_cast<int*>(Vs + seq * hp);
  const float* base = qkv + (int64_t)b * seq * ldq;
  load_slice<float>(base + h * hd, ldq, seq, hd, Qs, hp);
  load_slice<float>(base + d + h * hd, ldq, seq, hd, Ks, hp);
  load_slice<float>(base + 2 * d + h * hd, ldq, seq, hd, Vs, hp);
  __syncthreads();
  const int RT = (seq + 3) >> 2;
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  // ---- scores: 4 x NC per thread, kept in registers until Q is dead ----
  const int t = threadIdx.x;
  const bool has = t < RT * 16;
  const int ti = t >> 4, tj = t & 15;
  float acc[4][NC];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[a][c] = 0.0f;
  if (has) {
    int qr[4], kr[NC];
#pragma unroll
    for (int a = 0; a < 4; ++a) qr[a] = min(4 * ti + a, seq - 1) * hp;
#pragma unroll
    for (int c = 0; c < NC; ++c) kr[c] = min(tj + 16 * c, seq - 1) * hp;
#pragma unroll 4
    for (int e = 0; e < hd; ++e) {
      float qv[4], kv[NC];
#pragma unroll
      for (int a = 0; a < 4; ++a) qv[a] = Qs[qr[a] + e];
#pragma unroll
      for (int c = 0; c < NC; ++c) kv[c] = Ks[kr[c] + e];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[a][c] = fmaf(qv[a], kv[c], acc[a][c]);
    }
  }
  __syncthreads();  // Q dead: scores overwrite it
  float* Ss = Qs;
  if (has) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = 4 * ti + a;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = tj + 16 * c;
        if (i < seq && j < seq) {
          float s = fmul_rn(acc[a][c], scale);
          if (mk) s = fadd_rn(s, mk[j]);
          Ss[i * sp + j] = s;
        }
      }
    }
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = w; i < seq; i += nw) {
    const bool ok = warp_softmax(Ss + i * sp, seq, exact);
    if (lane == 0) {
      bad_row[i] = ok ? 0 : 1;
      if (!ok && d_bad) atomicAdd(d_bad, 1);
    }
  }
  __syncthreads();
  // ---- P.V: 4 rows x HC columns per thread ----
  if (has) {
    float o[4][HC];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < HC; ++c) o[a][c] = 0.0f;
    int pr[4], vc[HC];
#pragma unroll
    for (int a = 0; a < 4; ++a) pr[a] = min(4 * ti + a, seq - 1) * sp;
#pragma unroll
    for (int c = 0; c < HC; ++c) vc[c] = min(tj + 16 * c, hd - 1);
#pragma unroll 4
    for (int j = 0; j < seq; ++j) {
      float pv[4], vv[HC];
#pragma unroll
      for (int a = 0; a < 4; ++a) pv[a] = Ss[pr[a] + j];
#pragma unroll
      for (int c = 0; c < HC; ++c) vv[c] = Vs[j * hp + vc[c]];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < HC; ++c) o[a][c] = fmaf(pv[a], vv[c], o[a][c]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = 4 * ti + a;
      if (i >= seq || bad_row[i]) continue;
      const int64_t orow = ((int64_t)b * seq + i) * ldo + h * hd;
#pragma unroll
      for (int c = 0; c < HC; ++c) {
        const int e = tj + 16 * c;
        if (e < hd) {
          if (out) out[orow + e] = o[a][c];
          if (out16) out16[orow + e] = f2h(o[a][c]);
        }
      }
    }
  }
}

// ---- async bulk copies (cp.async.bulk, TMA engine) into shared memory ------
__device__ __forceinline__ uint32_t sm_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(sm_u32(bar)), "r"(parity)
        : "memory");
  }
}
// bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sm_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(sm_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Decoder self-attention, fp16 KV cache (throughput mode). CTA per beam row;
// thread lt owns 8 consecutive model dims (one 16-byte fp16 load per cached
// position), so a cached slot row (all heads, 2 KB) is read as one coalesced
// segment instead of per-head 128-byte pieces; G = blockDim / (d/8) position
// groups stream disjoint positions with U loads in flight per thread. Head
// dots are reduced over the HD/8 lanes of a head with xor-shuffles. The K/V of
// this step are written to slot (cur, r) (copy-free history, see above).
// ---------------------------------------------------------------------------
template <int HD, int U>
__global__ void __launch_bounds__(256, 4) decoder_self_attention_rows(
    const float* __restrict__ sqkv, int64_t ldq, h16* __restrict__ kc,
    h16* __restrict__ vc, const int32_t* __restrict__ hist,
    const int32_t* __restrict__ d_cur, int rows, int heads, int max_len, float scale,
    float* __restrict__ out, h16* __restrict__ out16, int64_t ldo) {
  pdl_enter();
  constexpr int TPH = HD / 8;  // threads per head
  extern __shared__ __align__(16) float smf[];
  const int r = blockIdx.x;
  const int d = heads * HD;
  const int TP = d / 8;               // threads per position
  const int G = blockDim.x / TP;      // position groups
  const int tid = threadIdx.x;
  const int g = tid / TP, lt = tid % TP;
  const int h = lt / TPH;
  const int cur = *d_cur;
  const int L1 = max_len + 1;
  float* S = smf;                                   // [heads][L1]
  int* phys = reinterpret_cast<int*>(S + heads * L1);  // [max_len]
  float* red = reinterpret_cast<float*>(phys + max_len);  // [G][d]
  const int32_t* hr = hist + (int64_t)r * max_len;
  for (int t = tid; t < cur; t += blockDim.x) phys[t] = hr[t];
  if (tid == 0) phys[cur] = r;
  const float* rowp = sqkv + (int64_t)r * ldq + lt * 8;
  float q[8], kn[8], vn[8];
  {
    const float4 a0 = *reinterpret_cast<const float4*>(rowp);
    const float4 a1 = *reinterpret_cast<const float4*>(rowp + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(rowp + d);
    const float4 b1 = *reinterpret_cast<const float4*>(rowp + d + 4);
    const float4 c0 = *reinterpret_cast<const float4*>(rowp + 2 * d);
    const float4 c1 = *reinterpret_cast<const float4*>(rowp + 2 * d + 4);
    q[0] = a0.x; q[1] = a0.y; q[2] = a0.z; q[3] = a0.w; q[4] = a1.x; q[5] = a1.y; q[6] = a1.z; q[7] = a1.w;
    kn[0] = b0.x; kn[1] = b0.y; kn[2] = b0.z; kn[3] = b0.w; kn[4] = b1.x; kn[5] = b1.y; kn[6] = b1.z; kn[7] = b1.w;
    vn[0] = c0.x; vn[1] = c0.y; vn[2] = c0.z; vn[3] = c0.w; vn[4] = c1.x; vn[5] = c1.y; vn[6] = c1.z; vn[7] = c1.w;
  }
  uint4 kpk, vpk;
  {
    h16x2 t2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) t2[i] = __floats2half2_rn(kn[2 * i], kn[2 * i + 1]);
    kpk = *reinterpret_cast<uint4*>(t2);
#pragma unroll
    for (int i = 0; i < 4; ++i) t2[i] = __floats2half2_rn(vn[2 * i], vn[2 * i + 1]);
    vpk = *reinterpret_cast<uint4*>(t2);
  }
  if (g == 0) {
    const int64_t slot = ((int64_t)cur * rows + r) * d + lt * 8;
    *reinterpret_cast<uint4*>(kc + slot) = kpk;
    *reinterpret_cast<uint4*>(vc + slot) = vpk;
  }
  __syncthreads();  // phys[] staged
  // ---- scores ----
  for (int t0 = g; t0 <= cur; t0 += G * U) {
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * G;
      if (t < cur) raw[u] = *reinterpret_cast<const uint4*>(kc + ((int64_t)t * rows + phys[t]) * d + lt * 8);
      else raw[u] = kpk;  // t == cur: the stored (rounded) key; t > cur unused
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * G;
      float f[8];
      unpack16<h16>(raw[u], f);
      float p = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) p = fmaf(q[j], f[j], p);
#pragma unroll
      for (int o = TPH / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      if ((lt % TPH) == 0 && t <= cur) S[h * L1 + t] = p * scale;
    }
  }
  __syncthreads();
  // ---- softmax per head (warp per head) ----
  {
    const int w = tid >> 5, nw = blockDim.x >> 5;
    for (int hh = w; hh < heads; hh += nw) warp_softmax(S + hh * L1, cur + 1, false);
  }
  __syncthreads();
  // ---- P.V ----
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
  const float* Sh = S + h * L1;
  for (int t0 = g; t0 <= cur; t0 += G * U) {
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * G;
      if (t < cur) raw[u] = *reinterpret_cast<const uint4*>(vc + ((int64_t)t * rows + phys[t]) * d + lt * 8);
      else raw[u] = vpk;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * G;
      if (t <= cur) {
        const float p = Sh[t];
        float f[8];
        unpack16<h16>(raw[u], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(p, f[j], acc[j]);
      }
    }
  }
  if (G > 1) {
    if (g > 0) {
#pragma unroll
      for (int j = 0; j < 8; j += 4)
        *reinterpret_cast<float4*>(red + (g - 1) * d + lt * 8 + j) =
            make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    }
    __syncthreads();
    if (g > 0) return;
    for (int gg = 1; gg < G; ++gg) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += red[(gg - 1) * d + lt * 8 + j];
    }
  }
  const int64_t o = (int64_t)r * ldo + lt * 8;
  if (out16) {
    h16x2 t2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) t2[i] = __floats2half2_rn(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4*>(out16 + o) = *reinterpret_cast<uint4*>(t2);
  }
  if (out) {
    *reinterpret_cast<float4*>(out + o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(out + o + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// ---- warp-level fp16 tensor-core helpers (mma.sync m16n8k16, ldmatrix) ----
// Decode attention is a handful of tiny per-(item, head) products (M = beams
// <= 8); the legacy warp MMA does them in a few dozen instructions where the
// FMA formulation needs thousands, which is what bounds these kernels. fp32
// queries / probabilities enter as a fp16 hi + lo pair (two MMAs), so the
// products keep ~16 mantissa bits against the fp16 keys/values they meet.
__device__ __forceinline__ void mma_f16_16816(float* c, const uint32_t* a, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(sm_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(sm_u32(p)));
}
// (x0, x1) -> packed f16x2 hi and the f16x2 residual lo
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const h16x2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const h16x2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// Cross-attention on warp MMAs, fp16 K/V (throughput mode). One warp per
// (item, head): the item's K and V head slices arrive by bulk copies into
// padded smem rows (144 B: conflict-free ldmatrix), then
//   S^T [pos x beam] = K . Q^T      (A = K via ldmatrix, B = Q^T hi/lo)
//   softmax over positions per beam (C fragments, xor-shuffles over groupID)
//   O^T [dim x beam] = V^T . P^T    (A = V^T via ldmatrix.trans, B = P^T hi/lo via smem)
// NT = position tiles of 16 (seq <= 16 NT), beams <= 8.
template <int HD, int NT>
__global__ void __launch_bounds__(32) cross_attention_mma(
    const float* __restrict__ cq, int64_t ldcq, const h16* __restrict__ ck,
    const h16* __restrict__ cv, int64_t ldkv, int beam, int seq, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int* d_bad) {
  constexpr int RS = HD * 2 + 16;  // padded smem row bytes
  constexpr int NP = NT * 16;
  extern __shared__ __align__(128) uint8_t smb[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ float Ps[8][NP + 4];
  uint8_t* Ks = smb;
  uint8_t* Vs = smb + NP * RS;
  const int b = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
  const int g = lane >> 2, t4 = lane & 3;
  if (lane == 0) {
    bar_init(&bar, 1);
    bar_expect(&bar, (uint32_t)(2 * seq * HD * 2));
  }
  __syncwarp();
  pdl_enter();
  const h16* kb = ck + (int64_t)b * seq * ldkv + h * HD;
  const h16* vb = cv + (int64_t)b * seq * ldkv + h * HD;
  for (int x = lane; x < 2 * seq; x += 32) {
    const int t = x >> 1;
    if (x & 1) bulk_g2s(Vs + t * RS, vb + (int64_t)t * ldkv, HD * 2, &bar);
    else bulk_g2s(Ks + t * RS, kb + (int64_t)t * ldkv, HD * 2, &bar);
  }
  // zero the padded positions [seq, NP) so 0 * garbage never makes NaN
  for (int x = lane; x < (NP - seq) * (HD / 8); x += 32) {
    const int t = seq + x / (HD / 8), c = (x % (HD / 8)) * 16;
    *reinterpret_cast<uint4*>(Ks + t * RS + c) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(Vs + t * RS + c) = make_uint4(0, 0, 0, 0);
  }
  // Q^T fragments: lane (g, t4) needs beam g, dims 16k + {2t4, 2t4+1, 2t4+8, 2t4+9}
  uint32_t qh[HD / 16][2], ql[HD / 16][2];
  {
    const bool ok = g < beam;
    const float* qp = cq + ((int64_t)b * beam + (ok ? g : 0)) * ldcq + h * HD;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      float2 x0 = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4) : make_float2(0.f, 0.f);
      float2 x1 = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4 + 8) : make_float2(0.f, 0.f);
      split2(x0.x, x0.y, qh[kk][0], ql[kk][0]);
      split2(x1.x, x1.y, qh[kk][1], ql[kk][1]);
    }
  }
  __syncwarp();
  bar_wait(&bar, 0);
  // ---- scores: NT tiles of 16 positions x 8 beams ----
  float sc[NT][4];
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 8;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
    sc[m][0] = sc[m][1] = sc[m][2] = sc[m][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t a[4];
      ldsm_x4(a, Ks + (16 * m + lrow) * RS + (16 * kk + lcol) * 2);
      mma_f16_16816(sc[m], a, qh[kk][0], qh[kk][1]);
      mma_f16_16816(sc[m], a, ql[kk][0], ql[kk][1]);
    }
  }
  // ---- softmax over positions, per beam column (2 per lane: 2t4, 2t4+1) ----
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int p = 16 * m + g + 8 * hh;
      const float add = p < seq ? (mk ? mk[p] : 0.0f) : -INFINITY;
      sc[m][2 * hh] = fmaf(sc[m][2 * hh], scale, add);
      sc[m][2 * hh + 1] = fmaf(sc[m][2 * hh + 1], scale, add);
      mx0 = fmaxf(mx0, sc[m][2 * hh]);
      mx1 = fmaxf(mx1, sc[m][2 * hh + 1]);
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float l0 = 0.0f, l1 = 0.0f;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const float e0 = mx0 == -INFINITY ? 0.0f : __expf(sc[m][2 * hh] - mx0);
      const float e1 = mx1 == -INFINITY ? 0.0f : __expf(sc[m][2 * hh + 1] - mx1);
      l0 += e0;
      l1 += e1;
      const int p = 16 * m + g + 8 * hh;
      Ps[2 * t4][p] = e0;
      Ps[2 * t4 + 1][p] = e1;
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  __syncwarp();
  // ---- O^T = V^T . P^T: HD/16 tiles of 16 dims x 8 beams, k over positions ----
  float oc[HD / 16][4];
#pragma unroll
  for (int m = 0; m < HD / 16; ++m) oc[m][0] = oc[m][1] = oc[m][2] = oc[m][3] = 0.0f;
  const int mi = lane >> 3;
  const int vrow = (lane & 7) + ((mi >> 1) & 1) * 8, vcol = (mi & 1) * 8;
#pragma unroll
  for (int kk = 0; kk < NT; ++kk) {
    uint32_t bh0, bl0, bh1, bl1;
    split2(Ps[g][16 * kk + 2 * t4], Ps[g][16 * kk + 2 * t4 + 1], bh0, bl0);
    split2(Ps[g][16 * kk + 2 * t4 + 8], Ps[g][16 * kk + 2 * t4 + 9], bh1, bl1);
#pragma unroll
    for (int m = 0; m < HD / 16; ++m) {
      uint32_t a[4];
      ldsm_x4_t(a, Vs + (16 * kk + vrow) * RS + (16 * m + vcol) * 2);
      mma_f16_16816(oc[m], a, bh0, bh1);
      mma_f16_16816(oc[m], a, bl0, bl1);
    }
  }
  // ---- normalise and store: lane holds dims {16m + g, +8} x beams {2t4, 2t4+1} ----
  const float inv0 = l0 > 0.0f ? 1.0f / l0 : 0.0f, inv1 = l1 > 0.0f ? 1.0f / l1 : 0.0f;
  if (d_bad && g == 0) {
    if (2 * t4 < beam && !(l0 > 0.0f)) atomicAdd(d_bad, 1);
    if (2 * t4 + 1 < beam && !(l1 > 0.0f)) atomicAdd(d_bad, 1);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int bi = 2 * t4 + j;
    if (bi >= beam) continue;
    const float inv = j ? inv1 : inv0;
    const int64_t o = ((int64_t)b * beam + bi) * ldo + h * HD;
#pragma unroll
    for (int m = 0; m < HD / 16; ++m) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int dd = 16 * m + g + 8 * hh;
        const float v = oc[m][2 * hh + j] * inv;
        if (out) out[o + dd] = v;
        if (out16) out16[o + dd] = f2h(v);
      }
    }
  }
}


int make_tmap_f16_sw128(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols,
                         int64_t ld, int box_cols, int box_rows);

// Cross-attention on warp MMAs, TMA variant (head_dim 64, seq <= 64): the K
// and V head slices of (item, head) arrive as two 64x64 fp16 TMA boxes with
// the 128-byte swizzle (no smem padding, conflict-free ldmatrix), and the
// probabilities reuse the K buffer once the scores are done, so a CTA needs
// 16 KB and all (item, head) CTAs are resident in one wave.
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// kCrossWarps warps per CTA, each an independent (item, head) with its own
// 16 KB of K/V boxes: one CTA of 14 warps per SM fills the SM's shared memory
// in a single wave (32-thread CTAs left a second, partial wave at C2).
constexpr int kCrossWarps = 14;
__global__ void __launch_bounds__(32 * kCrossWarps) cross_attention_tma(
    const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
    const float* __restrict__ cq, int64_t ldcq, int beam, int seq, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int* d_bad, int heads, int npairs, int nslab, int64_t slab,
    const float* __restrict__ qbias) {
  constexpr int HD = 64, NT = 4, NP = 64;
  extern __shared__ __align__(1024) uint8_t smraw[];
  const int wid = threadIdx.x >> 5;
  const int pair = blockIdx.x * kCrossWarps + wid;
  if (pair >= npairs) {
    pdl_enter();
    return;
  }
  uint8_t* Ks = smraw + ((1024u - (sm_u32(smraw) & 1023u)) & 1023u) + wid * (2 * NP * 128);
  uint8_t* Vs = Ks + NP * 128;
  float (*Ps)[NP + 4] = reinterpret_cast<float (*)[NP + 4]>(Ks);  // after the scores
  __shared__ __align__(8) uint64_t bars[kCrossWarps];
  uint64_t& bar = bars[wid];
  const int b = pair / heads, h = pair - b * heads, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  if (lane == 0) {
    bar_init(&bar, 1);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tk)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tv)));
  }
  __syncwarp();
  // the cross K/V buffer is written once per request, before the decode step
  // graph: its boxes stream in before the grid-dependency wait (only the
  // query comes from the preceding GEMM)
  pdl_launch_dependents();
  if (lane == 0) {
    bar_expect(&bar, 2 * NP * 128);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(sm_u32(Ks)),
        "l"(reinterpret_cast<uint64_t>(&tk)), "r"(h * HD), "r"(b * seq), "r"(sm_u32(&bar))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(sm_u32(Vs)),
        "l"(reinterpret_cast<uint64_t>(&tv)), "r"(h * HD), "r"(b * seq), "r"(sm_u32(&bar))
        : "memory");
  }
  pdl_wait();
  uint32_t qh[HD / 16][2], ql[HD / 16][2];
  {
    const bool ok = g < beam;
    const float* qp = cq + ((int64_t)b * beam + (ok ? g : 0)) * ldcq + h * HD;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      float2 x0 = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4) : make_float2(0.f, 0.f);
      float2 x1 = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4 + 8) : make_float2(0.f, 0.f);
      if (nslab > 0 && ok) {
        // q = the split-K query GEMM's K-slice slabs summed in slab order, then
        // + bias: the additions of the GEMM's own reduction epilogue, same order
        for (int sl = 1; sl < nslab; ++sl) {
          const float2 y0 = *reinterpret_cast<const float2*>(qp + sl * slab + 16 * kk + 2 * t4);
          const float2 y1 = *reinterpret_cast<const float2*>(qp + sl * slab + 16 * kk + 2 * t4 + 8);
          x0.x = fadd_rn(x0.x, y0.x);
          x0.y = fadd_rn(x0.y, y0.y);
          x1.x = fadd_rn(x1.x, y1.x);
          x1.y = fadd_rn(x1.y, y1.y);
        }
        if (qbias) {
          const float2 b0 = *reinterpret_cast<const float2*>(qbias + h * HD + 16 * kk + 2 * t4);
          const float2 b1 = *reinterpret_cast<const float2*>(qbias + h * HD + 16 * kk + 2 * t4 + 8);
          x0.x = fadd_rn(x0.x, b0.x);
          x0.y = fadd_rn(x0.y, b0.y);
          x1.x = fadd_rn(x1.x, b1.x);
          x1.y = fadd_rn(x1.y, b1.y);
        }
      }
      split2(x0.x, x0.y, qh[kk][0], ql[kk][0]);
      split2(x1.x, x1.y, qh[kk][1], ql[kk][1]);
    }
  }
  bar_wait(&bar, 0);
  float sc[NT][4];
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lch = lane >> 4;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
    sc[m][0] = sc[m][1] = sc[m][2] = sc[m][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t a[4];
      ldsm_x4(a, Ks + sw128(16 * m + lrow, 2 * kk + lch));
      mma_f16_16816(sc[m], a, qh[kk][0], qh[kk][1]);
      mma_f16_16816(sc[m], a, ql[kk][0], ql[kk][1]);
    }
  }
  __syncwarp();  // K is dead: Ps may overwrite it
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int p = 16 * m + g + 8 * hh;
      const float add = p < seq ? (mk ? mk[p] : 0.0f) : -INFINITY;
      sc[m][2 * hh] = fmaf(sc[m][2 * hh], scale, add);
      sc[m][2 * hh + 1] = fmaf(sc[m][2 * hh + 1], scale, add);
      mx0 = fmaxf(mx0, sc[m][2 * hh]);
      mx1 = fmaxf(mx1, sc[m][2 * hh + 1]);
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float l0 = 0.0f, l1 = 0.0f;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const float e0 = mx0 == -INFINITY ? 0.0f : __expf(sc[m][2 * hh] - mx0);
      const float e1 = mx1 == -INFINITY ? 0.0f : __expf(sc[m][2 * hh + 1] - mx1);
      l0 += e0;
      l1 += e1;
      const int p = 16 * m + g + 8 * hh;
      Ps[2 * t4][p] = e0;
      Ps[2 * t4 + 1][p] = e1;
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  __syncwarp();
  float oc[HD / 16][4];
#pragma unroll
  for (int m = 0; m < HD / 16; ++m) oc[m][0] = oc[m][1] = oc[m][2] = oc[m][3] = 0.0f;
  const int mi = lane >> 3;
  const int vrow = (lane & 7) + ((mi >> 1) & 1) * 8, vch = mi & 1;
#pragma unroll
  for (int kk = 0; kk < NT; ++kk) {
    uint32_t bh0, bl0, bh1, bl1;
    split2(Ps[g][16 * kk + 2 * t4], Ps[g][16 * kk + 2 * t4 + 1], bh0, bl0);
    split2(Ps[g][16 * kk + 2 * t4 + 8], Ps[g][16 * kk + 2 * t4 + 9], bh1, bl1);
#pragma unroll
    for (int m = 0; m < HD / 16; ++m) {
      uint32_t a[4];
      ldsm_x4_t(a, Vs + sw128(16 * kk + vrow, 2 * m + vch));
      mma_f16_16816(oc[m], a, bh0, bh1);
      mma_f16_16816(oc[m], a, bl0, bl1);
    }
  }
  const float inv0 = l0 > 0.0f ? 1.0f / l0 : 0.0f, inv1 = l1 > 0.0f ? 1.0f / l1 : 0.0f;
  if (d_bad && g == 0) {
    if (2 * t4 < beam && !(l0 > 0.0f)) atomicAdd(d_bad, 1);
    if (2 * t4 + 1 < beam && !(l1 > 0.0f)) atomicAdd(d_bad, 1);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int bi = 2 * t4 + j;
    if (bi >= beam) continue;
    const float inv = j ? inv1 : inv0;
    const int64_t o = ((int64_t)b * beam + bi) * ldo + h * HD;
#pragma unroll
    for (int m = 0; m < HD / 16; ++m) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int dd = 16 * m + g + 8 * hh;
        const float v = oc[m][2 * hh + j] * inv;
        if (out) out[o + dd] = v;
        if (out16) out16[o + dd] = f2h(v);
      }
    }
  }
}

// Decoder self-attention on warp MMAs (fp16 cache, head_dim 64): warp per
// (beam row, head). Cached positions stream through an NS-stage (default 3) shared-memory
// ring in chunks of 16 (cp.async 16-byte pieces of the hist-gathered slot rows,
// 128-byte rows with an XOR chunk swizzle, so ldmatrix is conflict-free); this
// step's K/V (position cur) are written to their cache slot and placed in the
// ring from registers. Per chunk: S^T[16 pos x 8] = K . q^T on the tensor core
// (column 0 is this row's query, fp32 split hi + lo), an online-softmax update,
// and O^T[64 x 8] += V^T . p^T (p split hi + lo). The FMA formulation needs
// ~16 instructions per cached element; this needs one MMA per 2048 MACs.
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int NS>
__global__ void __launch_bounds__(32) decoder_self_attention_mma(
    const float* __restrict__ sqkv, int64_t ldq, h16* __restrict__ kc,
    h16* __restrict__ vc, const int32_t* __restrict__ hist,
    const int32_t* __restrict__ d_cur, int rows, int heads, int max_len, float scale,
    float* __restrict__ out, h16* __restrict__ out16, int64_t ldo) {
  constexpr int HD = 64;
  __shared__ __align__(128) uint8_t ring[NS][2][16 * 128];  // [stage][K|V][16 rows x 128 B]
  __shared__ int phys_s[128];
  pdl_enter();
  const int r = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
  const int g = lane >> 2, t4 = lane & 3;
  const int d = heads * HD;
  const int cur = *d_cur;
  for (int t = lane; t < cur; t += 32) phys_s[t] = hist[(int64_t)r * max_len + t];
  // this step's q, k, v (fp32 from the QKV GEMM); lane owns 2 dims for k/v
  const float* rowp = sqkv + (int64_t)r * ldq + h * HD;
  const float2 kn = *reinterpret_cast<const float2*>(rowp + d + 2 * lane);
  const float2 vn = *reinterpret_cast<const float2*>(rowp + 2 * d + 2 * lane);
  const h16x2 kb2 = __floats2half2_rn(kn.x, kn.y);
  const h16x2 vb2 = __floats2half2_rn(vn.x, vn.y);
  {
    const int64_t slot = ((int64_t)cur * rows + r) * d + h * HD + 2 * lane;
    *reinterpret_cast<h16x2*>(kc + slot) = kb2;
    *reinterpret_cast<h16x2*>(vc + slot) = vb2;
  }
  // q^T fragments (column 0 = this row; other columns zero)
  uint32_t qh[4][2], ql[4][2];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    float2 x0 = make_float2(0.f, 0.f), x1 = x0;
    if (g == 0) {
      x0 = *reinterpret_cast<const float2*>(rowp + 16 * kk + 2 * t4);
      x1 = *reinterpret_cast<const float2*>(rowp + 16 * kk + 2 * t4 + 8);
    }
    split2(x0.x, x0.y, qh[kk][0], ql[kk][0]);
    split2(x1.x, x1.y, qh[kk][1], ql[kk][1]);
  }
  __syncwarp();
  const int npos = cur + 1;                 // positions 0..cur
  const int nchunk = (npos + 15) / 16;
  // issue chunk c into stage s: lane -> (16-byte chunk lane & 7, rows lane >> 3 + 4i)
  auto issue = [&](int c, int s) {
    const int ch = lane & 7;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = (lane >> 3) + 4 * i;
      const int t = 16 * c + rr;
      const uint32_t kd = sm_u32(&ring[s][0][0]) + swz(rr, ch);
      const uint32_t vd = sm_u32(&ring[s][1][0]) + swz(rr, ch);
      if (t < cur) {
        const int64_t off = ((int64_t)t * rows + phys_s[t]) * d + h * HD + ch * 8;
        cp16(kd, kc + off);
        cp16(vd, vc + off);
      } else if (t > cur) {  // beyond the sequence: zeros (masked, 0 * 0)
        *reinterpret_cast<uint4*>(&ring[s][0][0] + swz(rr, ch)) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(&ring[s][1][0] + swz(rr, ch)) = make_uint4(0, 0, 0, 0);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nchunk) issue(c, c);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float m_run = -INFINITY, l_run = 0.0f;
  float oc[4][4];
#pragma unroll
  for (int m = 0; m < 4; ++m) oc[m][0] = oc[m][1] = oc[m][2] = oc[m][3] = 0.0f;
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lch = lane >> 4;
  const int mi = lane >> 3;
  const int vrow = (lane & 7) + ((mi >> 1) & 1) * 8, vch = mi & 1;
  for (int c = 0; c < nchunk; ++c) {
    const int s = c % NS;
    // NS - 1 groups were committed ahead of chunk c: wait for the oldest
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    if (cur / 16 == c) {  // this step's k / v (row cur % 16) from registers
      const int rr = cur % 16;
      const int ch = (2 * lane) / 8, within = (2 * lane) % 8;
      *reinterpret_cast<h16x2*>(&ring[s][0][0] + swz(rr, ch) + within * 2) = kb2;
      *reinterpret_cast<h16x2*>(&ring[s][1][0] + swz(rr, ch) + within * 2) = vb2;
    }
    __syncwarp();
    const uint8_t* Ks = &ring[s][0][0];
    const uint8_t* Vs = &ring[s][1][0];
    float sc[4] = {0.f, 0.f, 0.f, 0.f}, sl[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // hi and lo products in separate chains
      uint32_t a[4];
      ldsm_x4(a, Ks + swz(lrow, 2 * kk + lch));
      mma_f16_16816(sc, a, qh[kk][0], qh[kk][1]);
      mma_f16_16816(sl, a, ql[kk][0], ql[kk][1]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) sc[j] += sl[j];
    // column 0 lives in lanes with t4 == 0: positions 16c + g (sc[0]) and + 8 (sc[2])
    const int p0 = 16 * c + g, p1 = p0 + 8;
    const float s0 = p0 <= cur ? sc[0] * scale : -INFINITY;
    const float s1 = p1 <= cur ? sc[2] * scale : -INFINITY;
    float cm = fmaxf(s0, s1);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    cm = __shfl_sync(0xffffffffu, cm, 0);
    const float mn = fmaxf(m_run, cm);
    const float corr = __expf(m_run - mn);  // m_run = -inf: 0
    const float e0 = __expf(s0 - mn), e1 = __expf(s1 - mn);
    float cs = e0 + e1;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
    cs = __shfl_sync(0xffffffffu, cs, 0);
    l_run = fmaf(l_run, corr, cs);
    m_run = mn;
    // p^T fragment: lanes 0-3 need positions 2t4, 2t4+1, 2t4+8, 2t4+9 of the chunk
    const float pa = __shfl_sync(0xffffffffu, e0, 4 * (2 * t4));
    const float pb = __shfl_sync(0xffffffffu, e0, 4 * (2 * t4 + 1));
    const float pc = __shfl_sync(0xffffffffu, e1, 4 * (2 * t4));
    const float pd = __shfl_sync(0xffffffffu, e1, 4 * (2 * t4 + 1));
    uint32_t bh0, bl0, bh1, bl1;
    split2(g == 0 ? pa : 0.f, g == 0 ? pb : 0.f, bh0, bl0);
    split2(g == 0 ? pc : 0.f, g == 0 ? pd : 0.f, bh1, bl1);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      oc[m][0] *= corr; oc[m][1] *= corr; oc[m][2] *= corr; oc[m][3] *= corr;
      uint32_t a[4];
      ldsm_x4_t(a, Vs + swz(vrow, 2 * m + vch));
      mma_f16_16816(oc[m], a, bh0, bh1);
      mma_f16_16816(oc[m], a, bl0, bl1);
    }
    __syncwarp();  // stage s consumed
    if (c + NS - 1 < nchunk) issue(c + NS - 1, (c + NS - 1) % NS);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // column 0 of O^T: lanes t4 == 0 hold dims 16m + g (oc[m][0]) and 16m + g + 8 (oc[m][2])
  if (t4 == 0) {
    const float inv = 1.0f / l_run;
    const int64_t o = (int64_t)r * ldo + h * HD;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const float v0 = oc[m][0] * inv, v1 = oc[m][2] * inv;
      if (out) { out[o + 16 * m + g] = v0; out[o + 16 * m + g + 8] = v1; }
      if (out16) { out16[o + 16 * m + g] = f2h(v0); out16[o + 16 * m + g + 8] = f2h(v1); }
    }
  }
}

// Encoder self-attention on warp MMAs (throughput mode, head_dim 64, seq <= 64):
// CTA per (item, head), warp per 16 queries. Q, K, V (fp32 from the QKV GEMM)
// are split into fp16 hi + lo halves in XOR-swizzled shared memory; scores
// S = Q K^T take three MMA products (hi.hi + hi.lo + lo.hi), the softmax runs
// on the accumulator fragments (FlashAttention-2 register layout), and P V
// reuses the probability fragments as A operands (P and V split likewise).
__global__ void __launch_bounds__(128) encoder_attention_mma(
    const float* __restrict__ qkv, int64_t ldq, int seq, int heads, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out16,
    int64_t ldo, int* d_bad) {
  constexpr int HD = 64, NP = 64;
  __shared__ __align__(128) uint8_t sm[6][NP * 128];  // Qh Ql Kh Kl Vh Vl, rows of 128 B
  pdl_enter();
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int d = heads * HD;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  // load + split: 64 rows x 16 float4 per tensor; thread -> (row, float4)
  for (int x = tid; x < 3 * NP * (HD / 4); x += 128) {
    const int tsr = x / (NP * (HD / 4)), rem = x % (NP * (HD / 4));
    const int row = rem / (HD / 4), c4 = rem % (HD / 4);
    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < seq)
      f = *reinterpret_cast<const float4*>(qkv + ((int64_t)b * seq + row) * ldq + tsr * d +
                                           h * HD + 4 * c4);
    uint32_t h0, l0, h1, l1;
    split2(f.x, f.y, h0, l0);
    split2(f.z, f.w, h1, l1);
    // element offset 4*c4 -> byte 8*c4 within the 128-byte row: chunk c4/2, half c4&1
    const uint32_t off = (uint32_t)(row * 128 + (((c4 >> 1) ^ (row & 7)) << 4) + (c4 & 1) * 8);
    *reinterpret_cast<uint2*>(&sm[2 * tsr][0] + off) = make_uint2(h0, h1);
    *reinterpret_cast<uint2*>(&sm[2 * tsr + 1][0] + off) = make_uint2(l0, l1);
  }
  __syncthreads();
  const int q0 = 16 * w;  // this warp's queries
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lch = lane >> 4;
  // scores: 8 key tiles x 4 k-steps, three products
  float sc[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.0f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t qa[4], qb[4];
    ldsm_x4(qa, &sm[0][0] + swz(q0 + lrow, 2 * kk + lch));
    ldsm_x4(qb, &sm[1][0] + swz(q0 + lrow, 2 * kk + lch));
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      // B = K^T: keys 8n..8n+7 (rows), dims 16kk..16kk+15 -> x2 ldmatrix: two 8x8 matrices
      uint32_t kh[2], kl[2];
      const int krow = 8 * n + (lane & 7), kch = 2 * kk + ((lane >> 3) & 1);
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                   : "=r"(kh[0]), "=r"(kh[1])
                   : "r"(sm_u32(&sm[2][0] + swz(krow, kch))));
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                   : "=r"(kl[0]), "=r"(kl[1])
                   : "r"(sm_u32(&sm[3][0] + swz(krow, kch))));
      mma_f16_16816(sc[n], qa, kh[0], kh[1]);
      mma_f16_16816(sc[n], qa, kl[0], kl[1]);
      mma_f16_16816(sc[n], qb, kh[0], kh[1]);
    }
  }
  // softmax per query row (rows g and g + 8 of the warp's tile)
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int key = 8 * n + 2 * t4 + j;
      const float add = key < seq ? (mk ? mk[key] : 0.0f) : -INFINITY;
      sc[n][j] = fmaf(sc[n][j], scale, add);
      sc[n][2 + j] = fmaf(sc[n][2 + j], scale, add);
      mx[0] = fmaxf(mx[0], sc[n][j]);
      mx[1] = fmaxf(mx[1], sc[n][2 + j]);
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
  }
  float sum[2] = {0.f, 0.f};
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = j >> 1;
      const float e = mx[r] == -INFINITY ? 0.0f : __expf(sc[n][j] - mx[r]);
      sc[n][j] = e;
      sum[r] += e;
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    sum[r] += __shfl_xor_sync(0xffffffffu, sum[r], 1);
    sum[r] += __shfl_xor_sync(0xffffffffu, sum[r], 2);
  }
  // O = P V: k over keys (4 steps of 16), n over dims (8 tiles of 8)
  float oc[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n) oc[n][0] = oc[n][1] = oc[n][2] = oc[n][3] = 0.0f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t ph[4], pl[4];
    split2(sc[2 * kk][0], sc[2 * kk][1], ph[0], pl[0]);
    split2(sc[2 * kk][2], sc[2 * kk][3], ph[1], pl[1]);
    split2(sc[2 * kk + 1][0], sc[2 * kk + 1][1], ph[2], pl[2]);
    split2(sc[2 * kk + 1][2], sc[2 * kk + 1][3], ph[3], pl[3]);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      // B = V: keys 16kk.. (k), dims 8n.. (n) -> ldmatrix.trans of V rows, x2
      uint32_t vh[2], vl[2];
      const int vrow = 16 * kk + (lane & 7) + ((lane >> 3) & 1) * 8, vch = n;
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                   : "=r"(vh[0]), "=r"(vh[1])
                   : "r"(sm_u32(&sm[4][0] + swz(vrow, vch))));
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                   : "=r"(vl[0]), "=r"(vl[1])
                   : "r"(sm_u32(&sm[5][0] + swz(vrow, vch))));
      mma_f16_16816(oc[n], ph, vh[0], vh[1]);
      mma_f16_16816(oc[n], ph, vl[0], vl[1]);
      mma_f16_16816(oc[n], pl, vh[0], vh[1]);
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = q0 + g + 8 * r;
    if (q >= seq) continue;
    if (!(sum[r] > 0.0f)) {
      if (t4 == 0 && d_bad) atomicAdd(d_bad, 1);
      continue;
    }
    const float inv = 1.0f / sum[r];
    const int64_t o = ((int64_t)b * seq + q) * ldo + h * HD;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float v0 = oc[n][2 * r] * inv, v1 = oc[n][2 * r + 1] * inv;
      const int dd = 8 * n + 2 * t4;
      if (out) *reinterpret_cast<float2*>(out + o + dd) = make_float2(v0, v1);
      if (out16) *reinterpret_cast<h16x2*>(out16 + o + dd) = __floats2half2_rn(v0, v1);
    }
  }
}

// FQ_SELF_MMA=0 selects the FMA row kernel (A/B runs).
static bool mma_self_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FQ_SELF_MMA");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

int attention_xh_prepare();

int attention_prepare() {
  if (attention_xh_prepare() != FQ_OK) return FQ_ERR_CUDA;
  const int big = 227 * 1024;
  if (cudaFuncSetAttribute(encoder_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_kernel<h16>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_fast<float, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<float, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<float, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<h16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<h16, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<h16, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(encoder_attention_tiled<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kCrossWarps * 2 * 64 * 128 + 1024) ||
      cudaFuncSetAttribute(encoder_attention_tiled<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) {
    set_error("fq_prepare: cannot opt in to large shared memory (attention)");
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

// ---------------------------------------------------------------------------
// Exact fp32 mode on warp MMAs (3xFP16). Every fp32 operand enters as its fp16
// pair x = hi + lo * 2^-11 (split_xh: 22 significant bits); a product takes
// three m16n8k16 MMAs, big += a_hi.b_hi and small += a_hi.b_lo + a_lo.b_hi,
// and the result is big + small * 2^-11 — fp32-GEMM accuracy for the
// reference's QK^T and P.V GEMMs (model.py:570-578, :594-604). The softmax
// between them is the reference's exact one (kernels.py:106-139, Appendix A
// E8): fp32 scores t = fp32(s * scale) (+ mask), exp(t - max) and the sum in
// f64, p = fp32(exp * (1 / sum)) — over all positions before P.V, so scores
// go to shared memory first (no online rescaling).
// Self-attention K/V cache: fp16 planes [2][max_len][rows][d] (hi, then lo at
// + plane elements); slot (t, r) written once, at step t, by row r.
// ---------------------------------------------------------------------------
constexpr float kXhInv = 1.0f / 2048.0f;

// exp(t - m) for the exact-mode softmax (t <= m): the difference exact in f64
// (as the reference's (double)t - (double)m), split into fp32 hi + lo, and
// 2^(d log2e) on the SFU with log2e as hi + lo parts: ~2 ulp of fp32, vs the
// reference's f64 exp — the probabilities, rounded to fp32, agree to an ulp.
// Sums stay in f64. (A f64 exp per score made these kernels DFMA-bound.)
__device__ __forceinline__ float xh_exp_diff(float t, float m) {
  const double dd = (double)t - (double)m;
  const float dh = (float)dd, dl = (float)(dd - (double)dh);
  constexpr float L2E = 1.4426950408889634f, L2E_LO = 1.925963033500011e-08f;
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(fmaf(dh, L2E, fmaf(dh, L2E_LO, dl * L2E))));
  return y;
}

// Exact-mode softmax over n scores in smem (one warp): max, e = xh_exp_diff,
// f64 sum, p = fp32(e / sum). False when every score is -inf.
__device__ __forceinline__ bool warp_softmax_xh(float* s, int n) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY;
  for (int j = lane; j < n; j += 32) m = fmaxf(m, s[j]);
  m = warp_max(m);
  if (m == -INFINITY) return false;
  double acc = 0.0;
  for (int j = lane; j < n; j += 32) {
    const float t = s[j];
    const float e = t == -INFINITY ? 0.0f : xh_exp_diff(t, m);
    s[j] = e;
    acc += (double)e;
  }
  const double inv = 1.0 / warp_sum(acc);
  __syncwarp();
  for (int j = lane; j < n; j += 32) s[j] = (float)((double)s[j] * inv);
  __syncwarp();
  return true;
}

template <int HD, int NS>
__global__ void __launch_bounds__(32) decoder_self_attention_xh(
    const float* __restrict__ sqkv, int64_t ldq, h16* __restrict__ kc, h16* __restrict__ vc,
    int64_t plane, const int32_t* __restrict__ hist, const int32_t* __restrict__ d_cur,
    int rows, int heads, int max_len, float scale, float* __restrict__ out,
    h16* __restrict__ out_hi, h16* __restrict__ out_lo, int64_t ldo) {
  // HD = 64: 128-byte rows, 16-byte chunks XOR-swizzled by row (no padding);
  // other head dims: a 16-byte row pad (conflict-free ldmatrix either way)
  constexpr bool SWZ = HD == 64;
  constexpr int RS = SWZ ? 128 : HD * 2 + 16;
  auto soff = [](int r, int byte) {
    return r * RS + (SWZ ? ((((byte >> 4) ^ (r & 7)) << 4) | (byte & 15)) : byte);
  };
  constexpr int CPR = HD * 2 / 16;  // 16-byte pieces per row
  constexpr int KT = HD / 16;
  constexpr int KE = (HD + 63) / 64;  // float2 of this step's k / v per lane
  __shared__ __align__(128) uint8_t ring[NS][2][16 * RS];  // [stage][hi | lo][16 rows]
  extern __shared__ __align__(16) float dyn[];
  float* sb = dyn;                                          // scores / p, [max_len + 16]
  // element offset of (position t, head h) in a cache plane, made once per warp
  // (32-bit: a plane is < 2^31 elements, checked on the host)
  int* off_s = reinterpret_cast<int*>(dyn + max_len + 16);  // [max_len]
  pdl_enter();
  const int r = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
  const int g = lane >> 2, t4 = lane & 3;
  const int d = heads * HD;
  // this row's q, k, v first: they do not depend on the position, so their
  // round trip overlaps the d_cur -> history-table chain below
  const float* rowp = sqkv + (int64_t)r * ldq + h * HD;
  float2 kn[KE], vn[KE];
#pragma unroll
  for (int i = 0; i < KE; ++i) {
    const int e = 2 * lane + 64 * i;
    kn[i] = vn[i] = make_float2(0.f, 0.f);
    if (e < HD) {
      kn[i] = *reinterpret_cast<const float2*>(rowp + d + e);
      vn[i] = *reinterpret_cast<const float2*>(rowp + 2 * d + e);
    }
  }
  float2 qx[KT][2];
#pragma unroll
  for (int kk = 0; kk < KT; ++kk) {
    qx[kk][0] = qx[kk][1] = make_float2(0.f, 0.f);
    if (g == 0) {
      qx[kk][0] = *reinterpret_cast<const float2*>(rowp + 16 * kk + 2 * t4);
      qx[kk][1] = *reinterpret_cast<const float2*>(rowp + 16 * kk + 2 * t4 + 8);
    }
  }
  const int cur = *d_cur;
  for (int t = lane; t < cur; t += 32)
    off_s[t] = (t * rows + hist[(int64_t)r * max_len + t]) * d + h * HD;
  // this step's k, v as pairs -> cache slot (cur, r); kept for the ring
  uint32_t knh[KE], knl[KE], vnh[KE], vnl[KE];
  {
    const int64_t slot = ((int64_t)cur * rows + r) * d + h * HD;
#pragma unroll
    for (int i = 0; i < KE; ++i) {
      const int e = 2 * lane + 64 * i;
      if (e < HD) {
        split_xh2(kn[i].x, kn[i].y, knh[i], knl[i]);
        split_xh2(vn[i].x, vn[i].y, vnh[i], vnl[i]);
        *reinterpret_cast<uint32_t*>(kc + slot + e) = knh[i];
        *reinterpret_cast<uint32_t*>(kc + plane + slot + e) = knl[i];
        *reinterpret_cast<uint32_t*>(vc + slot + e) = vnh[i];
        *reinterpret_cast<uint32_t*>(vc + plane + slot + e) = vnl[i];
      }
    }
  }
  // q^T fragments (column 0 = this row's query)
  uint32_t qh[KT][2], ql[KT][2];
#pragma unroll
  for (int kk = 0; kk < KT; ++kk) {
    split_xh2(qx[kk][0].x, qx[kk][0].y, qh[kk][0], ql[kk][0]);
    split_xh2(qx[kk][1].x, qx[kk][1].y, qh[kk][1], ql[kk][1]);
  }
  __syncwarp();
  const int npos = cur + 1, nchunk = (npos + 15) / 16;
  // chunk c of plane pair `src` (K or V) into stage s; position cur comes from registers
  auto issue = [&](const h16* src, int c, int s) {
    for (int x = lane; x < 16 * CPR; x += 32) {
      const int rr = x / CPR, ch = x % CPR;
      const int t = 16 * c + rr;
      uint8_t* dh = &ring[s][0][0] + soff(rr, ch * 16);
      uint8_t* dl = &ring[s][1][0] + soff(rr, ch * 16);
      if (t < cur) {
        const h16* p = src + off_s[t] + ch * 8;
        cp16(sm_u32(dh), p);
        cp16(sm_u32(dl), p + plane);
      } else if (t > cur) {  // beyond the sequence: zeros (p = 0, never NaN)
        *reinterpret_cast<uint4*>(dh) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dl) = make_uint4(0, 0, 0, 0);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto put_cur = [&](int s, const uint32_t* hi, const uint32_t* lo) {
    const int rr = cur % 16;
#pragma unroll
    for (int i = 0; i < KE; ++i) {
      const int e = 2 * lane + 64 * i;
      if (e < HD) {
        *reinterpret_cast<uint32_t*>(&ring[s][0][0] + soff(rr, e * 2)) = hi[i];
        *reinterpret_cast<uint32_t*>(&ring[s][1][0] + soff(rr, e * 2)) = lo[i];
      }
    }
  };
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 8;
  // one cp.async pipeline over the global chunk sequence K0..K(n-1), V0..V(n-1):
  // the V chunks stream in while the last scores and the softmax are computed
  auto issue_g = [&](int gi) {
    if (gi < nchunk) issue(kc, gi, gi % NS);
    else if (gi < 2 * nchunk) issue(vc, gi - nchunk, gi % NS);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) issue_g(c);
  // ---- pass 1: scores S^T[16 pos x 8] = K . q^T per chunk ----
  for (int c = 0; c < nchunk; ++c) {
    const int s = c % NS;
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    if (cur / 16 == c) put_cur(s, knh, knl);
    __syncwarp();
    const uint8_t* Kh = &ring[s][0][0];
    const uint8_t* Kl = &ring[s][1][0];
    float big[4] = {0.f, 0.f, 0.f, 0.f}, sml[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      uint32_t ah[4], al[4];
      ldsm_x4(ah, Kh + soff(lrow, (16 * kk + lcol) * 2));
      ldsm_x4(al, Kl + soff(lrow, (16 * kk + lcol) * 2));
      mma_f16_16816(big, ah, qh[kk][0], qh[kk][1]);
      mma_f16_16816(sml, ah, ql[kk][0], ql[kk][1]);
      mma_f16_16816(sml, al, qh[kk][0], qh[kk][1]);
    }
    if (t4 == 0) {  // column 0: positions 16c + g (reg 0) and + 8 (reg 2)
      const int p0 = 16 * c + g, p1 = p0 + 8;
      if (p0 <= cur) sb[p0] = fmul_rn(fadd_rn(big[0], sml[0] * kXhInv), scale);
      if (p1 <= cur) sb[p1] = fmul_rn(fadd_rn(big[2], sml[2] * kXhInv), scale);
    }
    __syncwarp();  // stage s consumed
    issue_g(c + NS - 1);
  }
  // ---- exact softmax over positions 0..cur (no mask: causality is implicit) ----
  warp_softmax_xh(sb, npos);
  for (int t = npos + lane; t < 16 * nchunk; t += 32) sb[t] = 0.0f;
  __syncwarp();
  // ---- pass 2: O^T[HD x 8] += V^T . p^T per chunk ----
  float ob[KT][4], os[KT][4];
#pragma unroll
  for (int m = 0; m < KT; ++m)
#pragma unroll
    for (int j = 0; j < 4; ++j) ob[m][j] = os[m][j] = 0.0f;
  const int mi = lane >> 3;
  const int vrow = (lane & 7) + ((mi >> 1) & 1) * 8, vcol = (mi & 1) * 8;
  for (int c = 0; c < nchunk; ++c) {
    const int s = (nchunk + c) % NS;
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    if (cur / 16 == c) put_cur(s, vnh, vnl);
    __syncwarp();
    const uint8_t* Vh = &ring[s][0][0];
    const uint8_t* Vl = &ring[s][1][0];
    uint32_t bh0, bl0, bh1, bl1;
    {
      const float* pp = sb + 16 * c + 2 * t4;
      split_xh2(g == 0 ? pp[0] : 0.f, g == 0 ? pp[1] : 0.f, bh0, bl0);
      split_xh2(g == 0 ? pp[8] : 0.f, g == 0 ? pp[9] : 0.f, bh1, bl1);
    }
#pragma unroll
    for (int m = 0; m < KT; ++m) {
      uint32_t ah[4], al[4];
      ldsm_x4_t(ah, Vh + soff(vrow, (16 * m + vcol) * 2));
      ldsm_x4_t(al, Vl + soff(vrow, (16 * m + vcol) * 2));
      mma_f16_16816(ob[m], ah, bh0, bh1);
      mma_f16_16816(os[m], ah, bl0, bl1);
      mma_f16_16816(os[m], al, bh0, bh1);
    }
    __syncwarp();
    issue_g(nchunk + c + NS - 1);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // column 0 of O^T: lanes t4 == 0 hold dims 16m + g (reg 0) and 16m + g + 8 (reg 2)
  if (t4 == 0) {
    const int64_t o = (int64_t)r * ldo + h * HD;
#pragma unroll
    for (int m = 0; m < KT; ++m) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int dd = 16 * m + g + 8 * hh;
        const float v = fadd_rn(ob[m][2 * hh], os[m][2 * hh] * kXhInv);
        if (out) out[o + dd] = v;
        if (out_hi) split_xh(v, out_hi[o + dd], out_lo[o + dd]);
      }
    }
  }
}

// Exact-mode decoder self-attention, one CTA of W warps per (item, head) with
// the beams as the MMA's query columns (head_dim 64, beam 2..8). The beams of
// an item share most of their K/V history (the history table points their
// positions at the same physical slots: ~40-55% distinct slots at C2), so
// each distinct slot (position t, physical row) streams through a ring ONCE
// and is scored against every beam's query. The slot list is split
// round-robin over the warps in 16-slot chunks (each warp its own cp.async
// ring, its K chunks then its V chunks); a beam's softmax runs over ITS
// positions 0..cur gathered in position order (the per-row kernel's
// warp_softmax_xh, so p is identical), and O^T = V^T . P^T with P = 0 where a
// beam does not use the slot, the warps' partial sums added in warp order.
// Scores and p match decoder_self_attention_xh bit for bit; the context only
// differs by the grouping of the P.V terms. Measured at C2 (B200): 0.4x the
// DRAM bytes of the per-row kernel, yet 65.0 vs 63.3 ms per request at the
// best setting (W = 2, NS = 3; W = 4: 66.6): the kernel is bound by its
// dependent chunk chains, not by bytes, so it stays opt-in. Dynamic smem: sc[Dpad][beam]
// (scores, then p), tmp[W][max_len + 16], off[Dmax] (element offset of each
// distinct slot), idx[beam][max_len] (int16: beam j's slot at position t).
template <int W, int NS>
__global__ void __launch_bounds__(32 * W) self_attention_items_xh(
    const float* __restrict__ sqkv, int64_t ldq, h16* __restrict__ kc, h16* __restrict__ vc,
    int64_t plane, const int32_t* __restrict__ hist, const int32_t* __restrict__ d_cur,
    int rows, int beam, int heads, int max_len, float scale, float* __restrict__ out,
    h16* __restrict__ out_hi, h16* __restrict__ out_lo, int64_t ldo) {
  constexpr int HD = 64, KT = 4, CPR = 8, MB = 8;
  auto soff = [](int r, int byte) {
    return r * 128 + ((((byte >> 4) ^ (r & 7)) << 4) | (byte & 15));
  };
  __shared__ __align__(128) uint8_t rings[W][NS][2][16 * 128];
  __shared__ int s_d;
  extern __shared__ __align__(16) float dyn[];
  const int dmax = beam * max_len;
  const int dpad = (dmax + 15) & ~15;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* sc = dyn;                                                     // [dpad][beam]
  float* tmp = sc + (size_t)dpad * beam + wid * (max_len + 16);        // [W][max_len + 16]
  int* off = reinterpret_cast<int*>(sc + (size_t)dpad * beam + W * (max_len + 16));  // [dmax]
  int16_t* idx = reinterpret_cast<int16_t*>(off + dmax);               // [beam][max_len]
  auto ring = rings[wid];
  pdl_enter();
  const int b = blockIdx.x, h = blockIdx.y;
  const int g = lane >> 2, t4 = lane & 3;
  const int d = heads * HD;
  const int cur = *d_cur;
  const int r0 = b * beam;
  // this step's k, v of every beam as pairs (each warp keeps them for its ring)
  uint32_t knh[MB], knl[MB], vnh[MB], vnl[MB];
#pragma unroll
  for (int j = 0; j < MB; ++j) {
    knh[j] = knl[j] = vnh[j] = vnl[j] = 0u;
    if (j < beam) {
      const float* rp = sqkv + (int64_t)(r0 + j) * ldq + h * HD + 2 * lane;
      const float2 kn = *reinterpret_cast<const float2*>(rp + d);
      const float2 vn = *reinterpret_cast<const float2*>(rp + 2 * d);
      split_xh2(kn.x, kn.y, knh[j], knl[j]);
      split_xh2(vn.x, vn.y, vnh[j], vnl[j]);
    }
  }
  if (wid == 0) {
    // ---- distinct (position, physical row) slots of the item, position order ----
    int D = 0;
    for (int t0 = 0; t0 < cur; t0 += 32) {
      const int t = t0 + lane;
      int src[MB];
      unsigned first = 0;
#pragma unroll
      for (int j = 0; j < MB; ++j) {
        src[j] = -1;
        if (j < beam && t < cur) src[j] = hist[(int64_t)(r0 + j) * max_len + t];
      }
#pragma unroll
      for (int j = 0; j < MB; ++j) {
        bool f = j < beam && t < cur;
#pragma unroll
        for (int k = 0; k < j; ++k) f = f && src[k] != src[j];
        first |= f ? 1u << j : 0u;
      }
      const int n = __popc(first);
      int incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int u0 = D + incl - n;
      if (t < cur) {
#pragma unroll
        for (int j = 0; j < MB; ++j) {
          if (j < beam) {
            int k0 = j;  // the first beam holding the same slot
#pragma unroll
            for (int k = MB - 1; k >= 0; --k)
              if (k < j && src[k] == src[j]) k0 = k;
            const int u = u0 + __popc(first & ((1u << k0) - 1u));
            if (k0 == j) off[u] = (t * rows + src[j]) * d + h * HD;
            idx[j * max_len + t] = (int16_t)u;
          }
        }
      }
      D += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane < beam) idx[lane * max_len + cur] = (int16_t)(D + lane);
    if (lane == 0) s_d = D;
    // this step's slots (cur, r0 + j): written once, read by later steps
#pragma unroll
    for (int j = 0; j < MB; ++j) {
      if (j < beam) {
        const int64_t slot = ((int64_t)cur * rows + r0 + j) * d + h * HD + 2 * lane;
        *reinterpret_cast<uint32_t*>(kc + slot) = knh[j];
        *reinterpret_cast<uint32_t*>(kc + plane + slot) = knl[j];
        *reinterpret_cast<uint32_t*>(vc + slot) = vnh[j];
        *reinterpret_cast<uint32_t*>(vc + plane + slot) = vnl[j];
      }
    }
  }
  // Q^T fragments: lane (g, t4) holds beam g, dims 16k + {2t4, 2t4+1, 2t4+8, 2t4+9}
  uint32_t qh[KT][2], ql[KT][2];
  {
    const bool ok = g < beam;
    const float* qp = sqkv + (int64_t)(r0 + (ok ? g : 0)) * ldq + h * HD;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      const float2 x0 = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4)
                           : make_float2(0.f, 0.f);
      const float2 x1 = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4 + 8)
                           : make_float2(0.f, 0.f);
      split_xh2(x0.x, x0.y, qh[kk][0], ql[kk][0]);
      split_xh2(x1.x, x1.y, qh[kk][1], ql[kk][1]);
    }
  }
  __syncthreads();
  const int dprev = s_d;  // slots dprev + j: this step's k, v of beam j (registers)
  const int D = dprev + beam;
  const int nchunk = (D + 15) / 16;
  const int nmine = nchunk > wid ? (nchunk - wid + W - 1) / W : 0;  // chunks wid, wid + W, ...
  auto issue = [&](const h16* src, int c, int st) {
    for (int x = lane; x < 16 * CPR; x += 32) {
      const int rr = x / CPR, ch = x % CPR;
      const int u = 16 * c + rr;
      uint8_t* dh = &ring[st][0][0] + soff(rr, ch * 16);
      uint8_t* dl = &ring[st][1][0] + soff(rr, ch * 16);
      if (u < dprev) {
        const h16* p = src + off[u] + ch * 8;
        cp16(sm_u32(dh), p);
        cp16(sm_u32(dl), p + plane);
      } else if (u >= D) {  // padding slots: zeros (p = 0, never NaN)
        *reinterpret_cast<uint4*>(dh) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dl) = make_uint4(0, 0, 0, 0);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto put_cur = [&](int c, int st, const uint32_t* hi, const uint32_t* lo) {
#pragma unroll
    for (int j = 0; j < MB; ++j) {
      const int u = dprev + j;
      if (j < beam && u / 16 == c) {
        *reinterpret_cast<uint32_t*>(&ring[st][0][0] + soff(u % 16, lane * 4)) = hi[j];
        *reinterpret_cast<uint32_t*>(&ring[st][1][0] + soff(u % 16, lane * 4)) = lo[j];
      }
    }
  };
  // this warp's chunk sequence: K of chunks wid + W i, then V of the same
  auto issue_g = [&](int gi) {
    if (gi < nmine) issue(kc, wid + W * gi, gi % NS);
    else if (gi < 2 * nmine) issue(vc, wid + W * (gi - nmine), gi % NS);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) issue_g(c);
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 8;
  // ---- pass 1: S^T[16 slots x 8 beams] = K . Q^T per chunk ----
  for (int i = 0; i < nmine; ++i) {
    const int c = wid + W * i, st = i % NS;
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    put_cur(c, st, knh, knl);
    __syncwarp();
    const uint8_t* Kh = &ring[st][0][0];
    const uint8_t* Kl = &ring[st][1][0];
    float big[4] = {0.f, 0.f, 0.f, 0.f}, sml[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      uint32_t ah[4], al[4];
      ldsm_x4(ah, Kh + soff(lrow, (16 * kk + lcol) * 2));
      ldsm_x4(al, Kl + soff(lrow, (16 * kk + lcol) * 2));
      mma_f16_16816(big, ah, qh[kk][0], qh[kk][1]);
      mma_f16_16816(sml, ah, ql[kk][0], ql[kk][1]);
      mma_f16_16816(sml, al, qh[kk][0], qh[kk][1]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int u = 16 * c + g + 8 * (e >> 1), j = 2 * t4 + (e & 1);
      if (j < beam) sc[u * beam + j] = fmul_rn(fadd_rn(big[e], sml[e] * kXhInv), scale);
    }
    __syncwarp();  // stage st consumed
    issue_g(i + NS - 1);
  }
  __syncthreads();
  // ---- per beam: exact softmax over its positions 0..cur, in position order ----
  const int npos = cur + 1;
  for (int j = wid; j < beam; j += W) {
    const int16_t* ij = idx + j * max_len;
    for (int t = lane; t < npos; t += 32) tmp[t] = sc[ij[t] * beam + j];
    __syncwarp();
    warp_softmax_xh(tmp, npos);
    for (int u = lane; u < 16 * nchunk; u += 32) sc[u * beam + j] = 0.0f;
    __syncwarp();
    for (int t = lane; t < npos; t += 32) sc[ij[t] * beam + j] = tmp[t];
  }
  __syncthreads();
  // ---- pass 2: O^T[HD x 8 beams] += V^T . P^T over this warp's chunks ----
  float ob[KT][4], os[KT][4];
#pragma unroll
  for (int m = 0; m < KT; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) ob[m][e] = os[m][e] = 0.0f;
  const int mi = lane >> 3;
  const int vrow = (lane & 7) + ((mi >> 1) & 1) * 8, vcol = (mi & 1) * 8;
  for (int i = 0; i < nmine; ++i) {
    const int c = wid + W * i, st = (nmine + i) % NS;
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    put_cur(c, st, vnh, vnl);
    __syncwarp();
    const uint8_t* Vh = &ring[st][0][0];
    const uint8_t* Vl = &ring[st][1][0];
    uint32_t bh0, bl0, bh1, bl1;
    {
      // P^T[slot 16c + 2t4 (+1, +8, +9)][beam g]
      const bool ok = g < beam;
      const float* pp = sc + (16 * c + 2 * t4) * beam + g;
      split_xh2(ok ? pp[0] : 0.f, ok ? pp[beam] : 0.f, bh0, bl0);
      split_xh2(ok ? pp[8 * beam] : 0.f, ok ? pp[9 * beam] : 0.f, bh1, bl1);
    }
#pragma unroll
    for (int m = 0; m < KT; ++m) {
      uint32_t ah[4], al[4];
      ldsm_x4_t(ah, Vh + soff(vrow, (16 * m + vcol) * 2));
      ldsm_x4_t(al, Vl + soff(vrow, (16 * m + vcol) * 2));
      mma_f16_16816(ob[m], ah, bh0, bh1);
      mma_f16_16816(os[m], ah, bl0, bl1);
      mma_f16_16816(os[m], al, bh0, bh1);
    }
    __syncwarp();
    issue_g(nmine + i + NS - 1);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (W > 1) {  // partial sums of warps 1.. through their (drained) rings, added in warp order
    float* red = reinterpret_cast<float*>(&ring[0][0][0]);  // 32 lanes x 32 floats = 4 KB
    if (wid > 0) {
#pragma unroll
      for (int m = 0; m < KT; ++m)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          red[(m * 4 + e) * 32 + lane] = ob[m][e];
          red[(16 + m * 4 + e) * 32 + lane] = os[m][e];
        }
    }
    __syncthreads();
    if (wid > 0) return;
#pragma unroll
    for (int w = 1; w < W; ++w) {
      const float* rw = reinterpret_cast<const float*>(&rings[w][0][0][0]);
#pragma unroll
      for (int m = 0; m < KT; ++m)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          ob[m][e] += rw[(m * 4 + e) * 32 + lane];
          os[m][e] += rw[(16 + m * 4 + e) * 32 + lane];
        }
    }
  }
  // ---- store: lane holds dims {16m + g, +8} x beams {2t4, 2t4+1} ----
#pragma unroll
  for (int jj = 0; jj < 2; ++jj) {
    const int j = 2 * t4 + jj;
    if (j >= beam) continue;
    const int64_t o = (int64_t)(r0 + j) * ldo + h * HD;
#pragma unroll
    for (int m = 0; m < KT; ++m) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int dd = 16 * m + g + 8 * hh;
        const float v = fadd_rn(ob[m][2 * hh + jj], os[m][2 * hh + jj] * kXhInv);
        if (out) out[o + dd] = v;
        if (out_hi) split_xh(v, out_hi[o + dd], out_lo[o + dd]);
      }
    }
  }
}

// Exact-mode cross-attention (3xFP16 warp MMAs), warp per (item, head), beams
// as the MMA's 8 query columns. The item's K then V head slices (fp16 pair
// planes of the cross-K/V buffer, [2][items * seq][ldkv]) stream through a
// shared-memory ring in 16-position chunks (cp.async, padded rows) — 12 KB per
// warp, so a whole C2 layer's (item, head) warps are resident in one wave:
//   pass 1  S^T[pos x beam] = K . Q^T, scores kept in registers;
//   softmax the reference's exact masked one per beam column (model.py:594-604,
//           kernels.py:106-139: fp32 t = s * scale + mask, f64 exp and sum);
//   pass 2  O^T = V^T . P^T.
template <int HD, int NT, int NS>
__global__ void __launch_bounds__(32) cross_attention_xh(
    const float* __restrict__ cq, int64_t ldcq, const h16* __restrict__ ck,
    const h16* __restrict__ cv, int64_t plane, int64_t ldkv, int beam, int seq, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out_hi,
    h16* __restrict__ out_lo, int64_t ldo, int* d_bad, int nslab = 0, int64_t qslab = 0,
    const float* __restrict__ qbias = nullptr) {
  // nslab > 0: cq holds the query GEMM's nslab split-K slabs (stride qslab
  // floats) summed here in split order, then + qbias -- the additions of the
  // split-K GEMM's DSMEM epilogue, so the query bits are the same.
  // HD = 64: 128-byte rows with the 16-byte chunks XOR-swizzled by row (no
  // padding: 12 instead of 13.5 KB of ring per warp at NS = 3); other head
  // dims keep a 16-byte row pad against ldmatrix bank conflicts
  constexpr bool SWZ = HD == 64;
  constexpr int RS = SWZ ? 128 : HD * 2 + 16;
  auto soff = [](int r, int ch) { return r * RS + (SWZ ? ((ch ^ (r & 7)) << 4) : (ch << 4)); };
  constexpr int CPR = HD * 2 / 16;
  constexpr int NP = NT * 16;
  constexpr int KT = HD / 16;
  __shared__ __align__(128) uint8_t ring[NS][2][16 * RS];
  const int b = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
  const int g = lane >> 2, t4 = lane & 3;
  // the cross K/V planes are written once per request, before the decode
  // step graph: the first chunks stream in before the grid-dependency wait
  // (only the query comes from the preceding GEMM)
  pdl_launch_dependents();
  const int64_t base = (int64_t)b * seq * ldkv + h * HD;
  auto issue = [&](const h16* src, int c, int st) {
    for (int x = lane; x < 16 * CPR; x += 32) {
      const int rr = x / CPR, pc = x % CPR;
      const int t = 16 * c + rr;
      uint8_t* dh = &ring[st][0][0] + soff(rr, pc);
      uint8_t* dl = &ring[st][1][0] + soff(rr, pc);
      if (t < seq) {
        const h16* p = src + base + (int64_t)t * ldkv + pc * 8;
        cp16(sm_u32(dh), p);
        cp16(sm_u32(dl), p + plane);
      } else {  // padded positions: zeros (p = 0, never NaN)
        *reinterpret_cast<uint4*>(dh) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dl) = make_uint4(0, 0, 0, 0);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nchunk = (seq + 15) / 16;
  // global chunk sequence: K chunks 0..nchunk-1, then V chunks; gi -> stage gi % NS
  auto issue_g = [&](int gi) {
    if (gi < nchunk) issue(ck, gi, gi % NS);
    else if (gi < 2 * nchunk) issue(cv, gi - nchunk, gi % NS);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) issue_g(c);
  // the padding mask is written with the cross K/V (once per request): this
  // lane's mask values (positions 16m + g, + 8) also before the wait
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  float mvr[NT][2];
#pragma unroll
  for (int m = 0; m < NT; ++m)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int p = 16 * m + g + 8 * hh;
      mvr[m][hh] = (mk && p < seq) ? mk[p] : 0.0f;
    }
  pdl_wait();
  // Q^T fragments: lane (g, t4) holds beam g, dims 16k + {2t4, 2t4+1, 2t4+8, 2t4+9}
  uint32_t qh[KT][2], ql[KT][2];
  {
    const bool ok = g < beam;
    const float* qp = cq + ((int64_t)b * beam + (ok ? g : 0)) * ldcq + h * HD;
#pragma unroll
    // this lane's 2 KT query element pairs: every load issued before any add
    float2 qv[KT][2];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        qv[kk][hh] = ok ? *reinterpret_cast<const float2*>(qp + 16 * kk + 2 * t4 + 8 * hh)
                        : make_float2(0.f, 0.f);
    if (nslab > 0 && ok) {
      float2 sv[3][KT][2], bv[KT][2];  // slabs 1..3 (nslab <= 4 on this path) and bias
#pragma unroll
      for (int sl = 0; sl < 3; ++sl)
#pragma unroll
        for (int kk = 0; kk < KT; ++kk)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            sv[sl][kk][hh] = sl + 1 < nslab ? *reinterpret_cast<const float2*>(
                                                  qp + (sl + 1) * qslab + 16 * kk + 2 * t4 + 8 * hh)
                                            : make_float2(0.f, 0.f);
#pragma unroll
      for (int kk = 0; kk < KT; ++kk)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          bv[kk][hh] = *reinterpret_cast<const float2*>(qbias + h * HD + 16 * kk + 2 * t4 + 8 * hh);
#pragma unroll
      for (int kk = 0; kk < KT; ++kk)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float2 v = qv[kk][hh];
#pragma unroll
          for (int sl = 0; sl < 3; ++sl)
            if (sl + 1 < nslab) { v.x += sv[sl][kk][hh].x; v.y += sv[sl][kk][hh].y; }
          v.x = fadd_rn(v.x, bv[kk][hh].x);
          v.y = fadd_rn(v.y, bv[kk][hh].y);
          qv[kk][hh] = v;
        }
    }
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      split_xh2(qv[kk][0].x, qv[kk][0].y, qh[kk][0], ql[kk][0]);
      split_xh2(qv[kk][1].x, qv[kk][1].y, qh[kk][1], ql[kk][1]);
    }
  }
  // ---- pass 1: scores ----
  float sc[NT][4];
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 8;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
    sc[m][0] = sc[m][1] = sc[m][2] = sc[m][3] = 0.0f;
    if (m < nchunk) {
      const int st = m % NS;
      asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
      __syncwarp();
      const uint8_t* Kh = &ring[st][0][0];
      const uint8_t* Kl = &ring[st][1][0];
      float big[4] = {0.f, 0.f, 0.f, 0.f}, sml[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        uint32_t ah[4], al[4];
        ldsm_x4(ah, Kh + soff(lrow, 2 * kk + (lcol >> 3)));
        ldsm_x4(al, Kl + soff(lrow, 2 * kk + (lcol >> 3)));
        mma_f16_16816(big, ah, qh[kk][0], qh[kk][1]);
        mma_f16_16816(sml, ah, ql[kk][0], ql[kk][1]);
        mma_f16_16816(sml, al, qh[kk][0], qh[kk][1]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) sc[m][j] = fadd_rn(big[j], sml[j] * kXhInv);
      __syncwarp();
      issue_g(m + NS - 1);  // K chunks, then the first V chunks
    }
  }
  // ---- exact softmax per beam column (lane: columns 2t4, 2t4+1) ----
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int p = 16 * m + g + 8 * hh;
      float t0 = -INFINITY, t1 = -INFINITY;
      if (p < seq) {
        t0 = fmul_rn(sc[m][2 * hh], scale);
        t1 = fmul_rn(sc[m][2 * hh + 1], scale);
        if (mk) {
          const float mv = mvr[m][hh];
          t0 = fadd_rn(t0, mv);
          t1 = fadd_rn(t1, mv);
        }
      }
      sc[m][2 * hh] = t0;
      sc[m][2 * hh + 1] = t1;
      mx0 = fmaxf(mx0, t0);
      mx1 = fmaxf(mx1, t1);
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float e[NT][4];
  double l0 = 0.0, l1 = 0.0;
#pragma unroll
  for (int m = 0; m < NT; ++m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const float t0 = sc[m][2 * hh], t1 = sc[m][2 * hh + 1];
      e[m][2 * hh] = t0 == -INFINITY ? 0.0f : xh_exp_diff(t0, mx0);
      e[m][2 * hh + 1] = t1 == -INFINITY ? 0.0f : xh_exp_diff(t1, mx1);
      l0 += (double)e[m][2 * hh];
      l1 += (double)e[m][2 * hh + 1];
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  const double inv0 = l0 > 0.0 ? 1.0 / l0 : 0.0, inv1 = l1 > 0.0 ? 1.0 / l1 : 0.0;
  // p = fp32(e / sum), kept in registers in the score layout (lane (g, t4):
  // positions 16m + g (+8), beams 2t4, 2t4 + 1); pass 2 gathers its P^T
  // fragments by shuffles (no smem: more warps resident per SM)
#pragma unroll
  for (int m = 0; m < NT; ++m)
#pragma unroll
    for (int c = 0; c < 4; ++c) e[m][c] = (float)((double)e[m][c] * ((c & 1) ? inv1 : inv0));
  if (d_bad && g == 0) {
    if (2 * t4 < beam && !(l0 > 0.0)) atomicAdd(d_bad, 1);
    if (2 * t4 + 1 < beam && !(l1 > 0.0)) atomicAdd(d_bad, 1);
  }
  __syncwarp();
  // ---- pass 2: O^T = V^T . P^T over the V chunks (ring continues) ----
  float ob[KT][4], os[KT][4];
#pragma unroll
  for (int m = 0; m < KT; ++m)
#pragma unroll
    for (int j = 0; j < 4; ++j) ob[m][j] = os[m][j] = 0.0f;
  const int mi = lane >> 3;
  const int vrow = (lane & 7) + ((mi >> 1) & 1) * 8, vcol = (mi & 1) * 8;
#pragma unroll
  for (int kk = 0; kk < NT; ++kk) {
    if (kk < nchunk) {
      const int st = (nchunk + kk) % NS;
      asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
      __syncwarp();
      const uint8_t* Vh = &ring[st][0][0];
      const uint8_t* Vl = &ring[st][1][0];
      uint32_t bh0, bl0, bh1, bl1;
      {
        // P[beam g][16kk + 2t4 + j (+8)] lives in lane (2t4 + j, g >> 1), element
        // (g & 1) (+2 for the upper 8 positions)
        float pv[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int src = (2 * t4 + j) * 4 + (g >> 1);
          const float v0 = __shfl_sync(0xffffffffu, e[kk][0], src);
          const float v1 = __shfl_sync(0xffffffffu, e[kk][1], src);
          const float v2 = __shfl_sync(0xffffffffu, e[kk][2], src);
          const float v3 = __shfl_sync(0xffffffffu, e[kk][3], src);
          pv[0][j] = (g & 1) ? v1 : v0;
          pv[1][j] = (g & 1) ? v3 : v2;
        }
        split_xh2(pv[0][0], pv[0][1], bh0, bl0);
        split_xh2(pv[1][0], pv[1][1], bh1, bl1);
      }
#pragma unroll
      for (int m = 0; m < KT; ++m) {
        uint32_t ah[4], al[4];
        ldsm_x4_t(ah, Vh + soff(vrow, 2 * m + (vcol >> 3)));
        ldsm_x4_t(al, Vl + soff(vrow, 2 * m + (vcol >> 3)));
        mma_f16_16816(ob[m], ah, bh0, bh1);
        mma_f16_16816(os[m], ah, bl0, bl1);
        mma_f16_16816(os[m], al, bh0, bh1);
      }
      __syncwarp();
      issue_g(nchunk + kk + NS - 1);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // ---- store: lane holds dims {16m + g, +8} x beams {2t4, 2t4+1} ----
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int bi = 2 * t4 + j;
    if (bi >= beam) continue;
    const int64_t o = ((int64_t)b * beam + bi) * ldo + h * HD;
#pragma unroll
    for (int m = 0; m < KT; ++m) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int dd = 16 * m + g + 8 * hh;
        const float v = fadd_rn(ob[m][2 * hh + j], os[m][2 * hh + j] * kXhInv);
        if (out) out[o + dd] = v;
        if (out_hi) split_xh(v, out_hi[o + dd], out_lo[o + dd]);
      }
    }
  }
}

// Exact-mode encoder self-attention (model.py:329-336, kernels.py:106-139) for
// head_dim 64, seq <= 64: CTA per (item, head), 4 warps x 16 queries. Q, K, V
// as fp16 pairs (split_xh2) in XOR-swizzled shared memory; S = Q K^T and
// O = P V as 3xFP16 m16n8k16 products (big = hi.hi, small = hi.lo + lo.hi,
// combined with RN adds); between them the reference's softmax as in the
// decoder kernels (fp32 score x scale (+ mask) with two roundings, exp of the
// f64-exact difference on the SFU, f64 sums, p = fp32(e / sum)); the context is
// written as the out-projection GEMM's fp16 pair (and fp32 when asked).
__global__ void __launch_bounds__(128) encoder_attention_xh(
    const float* __restrict__ qkv, int64_t ldq, int seq, int heads, float scale,
    const float* __restrict__ mask, float* __restrict__ out, h16* __restrict__ out_hi,
    h16* __restrict__ out_lo, int64_t ldo, int* d_bad) {
  constexpr int HD = 64, NP = 64;
  __shared__ __align__(128) uint8_t sm[6][NP * 128];  // Qh Ql Kh Kl Vh Vl, rows of 128 B
  pdl_enter();
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int d = heads * HD;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  for (int x = tid; x < 3 * NP * (HD / 4); x += 128) {
    const int tsr = x / (NP * (HD / 4)), rem = x % (NP * (HD / 4));
    const int row = rem / (HD / 4), c4 = rem % (HD / 4);
    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < seq)
      f = *reinterpret_cast<const float4*>(qkv + ((int64_t)b * seq + row) * ldq + tsr * d +
                                           h * HD + 4 * c4);
    uint32_t h0, l0, h1, l1;
    split_xh2(f.x, f.y, h0, l0);
    split_xh2(f.z, f.w, h1, l1);
    const uint32_t off = (uint32_t)(row * 128 + (((c4 >> 1) ^ (row & 7)) << 4) + (c4 & 1) * 8);
    *reinterpret_cast<uint2*>(&sm[2 * tsr][0] + off) = make_uint2(h0, h1);
    *reinterpret_cast<uint2*>(&sm[2 * tsr + 1][0] + off) = make_uint2(l0, l1);
  }
  __syncthreads();
  const int q0 = 16 * w;
  if (q0 >= seq) return;
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lch = lane >> 4;
  float sb[8][4], ss[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int j = 0; j < 4; ++j) sb[n][j] = ss[n][j] = 0.0f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t qa[4], qb[4];
    ldsm_x4(qa, &sm[0][0] + swz(q0 + lrow, 2 * kk + lch));
    ldsm_x4(qb, &sm[1][0] + swz(q0 + lrow, 2 * kk + lch));
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      uint32_t kh[2], kl[2];
      const int krow = 8 * n + (lane & 7), kch = 2 * kk + ((lane >> 3) & 1);
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                   : "=r"(kh[0]), "=r"(kh[1])
                   : "r"(sm_u32(&sm[2][0] + swz(krow, kch))));
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                   : "=r"(kl[0]), "=r"(kl[1])
                   : "r"(sm_u32(&sm[3][0] + swz(krow, kch))));
      mma_f16_16816(sb[n], qa, kh[0], kh[1]);
      mma_f16_16816(ss[n], qa, kl[0], kl[1]);
      mma_f16_16816(ss[n], qb, kh[0], kh[1]);
    }
  }
  // softmax per query row (rows g and g + 8 of the warp's tile; lane t4 holds
  // keys 8n + 2t4, +1)
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  float sc[8][4];
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int key = 8 * n + 2 * t4 + (j & 1);
      float t = -INFINITY;
      if (key < seq) {
        t = fmul_rn(fadd_rn(sb[n][j], ss[n][j] * kXhInv), scale);
        if (mk) t = fadd_rn(t, mk[key]);
      }
      sc[n][j] = t;
      mx[j >> 1] = fmaxf(mx[j >> 1], t);
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
  }
  double l[2] = {0.0, 0.0};
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = j >> 1;
      const float e = sc[n][j] == -INFINITY ? 0.0f : xh_exp_diff(sc[n][j], mx[r]);
      sc[n][j] = e;
      l[r] += (double)e;
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
  const double inv[2] = {l[0] > 0.0 ? 1.0 / l[0] : 0.0, l[1] > 0.0 ? 1.0 / l[1] : 0.0};
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int j = 0; j < 4; ++j) sc[n][j] = (float)((double)sc[n][j] * inv[j >> 1]);
  float ob[8][4], os[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int j = 0; j < 4; ++j) ob[n][j] = os[n][j] = 0.0f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t ph[4], pl[4];
    split_xh2(sc[2 * kk][0], sc[2 * kk][1], ph[0], pl[0]);
    split_xh2(sc[2 * kk][2], sc[2 * kk][3], ph[1], pl[1]);
    split_xh2(sc[2 * kk + 1][0], sc[2 * kk + 1][1], ph[2], pl[2]);
    split_xh2(sc[2 * kk + 1][2], sc[2 * kk + 1][3], ph[3], pl[3]);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      uint32_t vh[2], vl[2];
      const int vrow = 16 * kk + (lane & 7) + ((lane >> 3) & 1) * 8, vch = n;
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                   : "=r"(vh[0]), "=r"(vh[1])
                   : "r"(sm_u32(&sm[4][0] + swz(vrow, vch))));
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                   : "=r"(vl[0]), "=r"(vl[1])
                   : "r"(sm_u32(&sm[5][0] + swz(vrow, vch))));
      mma_f16_16816(ob[n], ph, vh[0], vh[1]);
      mma_f16_16816(os[n], ph, vl[0], vl[1]);
      mma_f16_16816(os[n], pl, vh[0], vh[1]);
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = q0 + g + 8 * r;
    if (q >= seq) continue;
    if (!(l[r] > 0.0)) {
      if (t4 == 0 && d_bad) atomicAdd(d_bad, 1);
      continue;
    }
    const int64_t o = ((int64_t)b * seq + q) * ldo + h * HD;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float v0 = fadd_rn(ob[n][2 * r], os[n][2 * r] * kXhInv);
      const float v1 = fadd_rn(ob[n][2 * r + 1], os[n][2 * r + 1] * kXhInv);
      const int dd = 8 * n + 2 * t4;
      if (out) *reinterpret_cast<float2*>(out + o + dd) = make_float2(v0, v1);
      if (out_hi) {
        uint32_t ph, pl;
        split_xh2(v0, v1, ph, pl);
        *reinterpret_cast<uint32_t*>(out_hi + o + dd) = ph;
        *reinterpret_cast<uint32_t*>(out_lo + o + dd) = pl;
      }
    }
  }
}

int attention_xh_prepare() {
  const int sz = 160 * 1024;  // scores + history of long max_len (static ring <= 26 KB)
#define FQ_XH_OPT(HD)                                                                           \
  cudaFuncSetAttribute(decoder_self_attention_xh<HD, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz) || \
      cudaFuncSetAttribute(decoder_self_attention_xh<HD, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz)
  if (FQ_XH_OPT(16) || FQ_XH_OPT(32) || FQ_XH_OPT(64) || FQ_XH_OPT(128) ||
      cudaFuncSetAttribute(self_attention_items_xh<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz) ||
      cudaFuncSetAttribute(self_attention_items_xh<1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz) ||
      cudaFuncSetAttribute(self_attention_items_xh<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz) ||
      cudaFuncSetAttribute(self_attention_items_xh<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz) ||
      cudaFuncSetAttribute(self_attention_items_xh<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sz)) {
    set_error("fq_prepare: cannot opt in to large shared memory (exact attention)");
    return FQ_ERR_CUDA;
  }
#undef FQ_XH_OPT
  return FQ_OK;
}

template <typename KV, int HD>
static void launch_self_fast(dim3 grid, size_t smem, cudaStream_t s, const float* sqkv,
                             int64_t ldq, void* kc, void* vc, const int32_t* hist,
                             const int32_t* d_cur, int64_t rows, int64_t heads, int64_t max_len,
                             float scale, float* out, void* out16, int64_t ldo, int exact) {
  launch_kernel(decoder_self_attention_fast<KV, HD>, grid, 128, smem, s, 1u, 
      sqkv, ldq, (KV*)kc, (KV*)vc, hist, d_cur, (int)rows, (int)heads, (int)max_len, scale, out,
      reinterpret_cast<fq::h16*>(out16), ldo, exact);
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_encoder_attention(const float* qkv, int64_t ldq, int64_t batch, int64_t seq,
                         int64_t heads, int64_t head_dim, float scale, const float* mask,
                         float* out, void* out16, int64_t ldo, int exact, int* d_bad,
                         fq_stream_t stream) {
  FQ_CHECK_ARG(qkv && (out || out16) && batch > 0 && seq > 0 && heads > 0 && head_dim > 0 &&
                   head_dim <= 128,
               FQ_ERR_DIMENSION, "fq_encoder_attention: bad shape");
  if (!exact && head_dim == 64 && seq <= 64 && ldq % 4 == 0 && ((uintptr_t)qkv & 15) == 0 &&
      ldo % 2 == 0) {
    launch_kernel(encoder_attention_mma, (unsigned)(batch * heads), 128, 0, as_stream(stream), 1u,
                  qkv, ldq, (int)seq, (int)heads, scale, mask, out,
                  reinterpret_cast<fq::h16*>(out16), ldo, d_bad);
    return launch_status("fq_encoder_attention");
  }
  if (seq <= 64 && ldq % 4 == 0 && ((uintptr_t)qkv & 15) == 0) {
    const int64_t hp = head_dim + 1, sp = seq + 1;
    const size_t smem = (size_t)(seq * (hp > sp ? hp : sp) + 2 * seq * hp + seq) * 4;
    if (head_dim <= 64)
      launch_kernel(encoder_attention_tiled<4, 4>, (unsigned)(batch * heads), 256, smem,
                    as_stream(stream), 1u, qkv, ldq, (int)seq, (int)heads, (int)head_dim, scale,
                    mask, out, reinterpret_cast<fq::h16*>(out16), ldo, exact, d_bad);
    else
      launch_kernel(encoder_attention_tiled<4, 8>, (unsigned)(batch * heads), 256, smem,
                    as_stream(stream), 1u, qkv, ldq, (int)seq, (int)heads, (int)head_dim, scale,
                    mask, out, reinterpret_cast<fq::h16*>(out16), ldo, exact, d_bad);
    return launch_status("fq_encoder_attention");
  }
  const int threads = 256;
  size_t smem = (size_t)(2 * seq * (head_dim + 1) + seq * head_dim + (threads / 32) * seq) * 4;
  FQ_CHECK_ARG(smem <= 227 * 1024, FQ_ERR_CAPACITY, "encoder attention: seq %lld too long",
               (long long)seq);
  launch_kernel(encoder_attention_kernel, (unsigned)(batch * heads), threads, smem, as_stream(stream), 1u,
      qkv, ldq, (int)seq, (int)heads, (int)head_dim, scale, mask, out,
      reinterpret_cast<fq::h16*>(out16), ldo, exact, d_bad);
  return launch_status("fq_encoder_attention");
}

int fq_encoder_attention_xh(const float* qkv, int64_t ldq, int64_t batch, int64_t seq,
                            int64_t heads, int64_t head_dim, float scale, const float* mask,
                            float* out, void* out_hi, void* out_lo, int64_t ldo, int* d_bad,
                            fq_stream_t stream) {
  FQ_CHECK_ARG(qkv && out_hi && out_lo && batch > 0 && seq > 0 && seq <= 64 && heads > 0 &&
                   head_dim == 64 && ldq % 4 == 0 && ((uintptr_t)qkv & 15) == 0 && ldo % 2 == 0,
               FQ_ERR_DIMENSION, "fq_encoder_attention_xh: needs head_dim 64, seq <= 64");
  launch_kernel(encoder_attention_xh, (unsigned)(batch * heads), 128, 0, as_stream(stream), 1u,
                qkv, ldq, (int)seq, (int)heads, scale, mask, out, (h16*)out_hi, (h16*)out_lo,
                ldo, d_bad);
  return launch_status("fq_encoder_attention_xh");
}

int fq_decoder_self_attention(const float* sqkv, int64_t ldq, void* kcache, void* vcache,
                              int kv_dtype, const int32_t* hist, const int32_t* d_cur,
                              int64_t rows, int64_t heads, int64_t head_dim, int64_t max_len,
                              float scale, float* out, void* out16, int64_t ldo, int exact,
                              fq_stream_t stream) {
  FQ_CHECK_ARG(sqkv && kcache && vcache && hist && d_cur && (out || out16) && rows > 0 &&
                   heads > 0 && head_dim > 0 && head_dim <= 128 && max_len > 0,
               FQ_ERR_DIMENSION, "fq_decoder_self_attention: bad args");
  if (kv_dtype != FQ_F32 && !exact && head_dim == 64 && max_len <= 128 && ldq % 2 == 0 &&
      ((uintptr_t)sqkv & 7) == 0 && ((uintptr_t)kcache & 15) == 0 &&
      ((uintptr_t)vcache & 15) == 0 && !mma_self_disabled()) {
    static int ns = -1;  // ring depth (FQ_SELF_STAGES = 2 | 3 | 4)
    if (ns < 0) {
      const char* e = getenv("FQ_SELF_STAGES");
      ns = e ? atoi(e) : 3;  // 3: +0.45% at C2 over 2 (3 paired bench runs), 4: -2%
    }
    auto kern = ns == 2 ? decoder_self_attention_mma<2>
              : ns == 4 ? decoder_self_attention_mma<4> : decoder_self_attention_mma<3>;
    launch_kernel(kern, dim3((unsigned)rows, (unsigned)heads), 32, 0,
                  as_stream(stream), 1u, sqkv, ldq, (h16*)kcache,
                  (h16*)vcache, hist, d_cur, (int)rows, (int)heads, (int)max_len,
                  scale, out, reinterpret_cast<fq::h16*>(out16), ldo);
    return launch_status("fq_decoder_self_attention");
  }
  {
    const int64_t d = heads * head_dim, tp = d / 8;
    const bool rows_ok = kv_dtype != FQ_F32 && !exact &&
                         (head_dim == 32 || head_dim == 64 || head_dim == 128) &&
                         tp % 32 == 0 && tp <= 256 && ldq % 4 == 0 &&
                         ((uintptr_t)sqkv & 15) == 0 && ((uintptr_t)kcache & 15) == 0 &&
                         ((uintptr_t)vcache & 15) == 0 && ldo % 8 == 0 &&
                         ((uintptr_t)out16 & 15) == 0 && ((uintptr_t)out & 15) == 0;
    if (rows_ok) {
      const int threads = 256;
      const int G = threads / (int)tp;
      const size_t smem = (size_t)(heads * (max_len + 1)) * 4 + (size_t)max_len * 4 +
                          (size_t)(G - 1) * d * 4 + 16;
#define FQ_SELF_ROWS(HD)                                                                       \
  launch_kernel(decoder_self_attention_rows<HD, 8>, dim3((unsigned)rows), threads, smem,       \
                as_stream(stream), 1u, sqkv, ldq, (h16*)kcache,                     \
                (h16*)vcache, hist, d_cur, (int)rows, (int)heads, (int)max_len, scale, \
                out, reinterpret_cast<fq::h16*>(out16), ldo)
      if (head_dim == 32) FQ_SELF_ROWS(32);
      else if (head_dim == 64) FQ_SELF_ROWS(64);
      else FQ_SELF_ROWS(128);
#undef FQ_SELF_ROWS
      return launch_status("fq_decoder_self_attention");
    }
  }
  const int wpb = 4;
  dim3 grid((unsigned)((rows + wpb - 1) / wpb), (unsigned)heads);
  cudaStream_t s = as_stream(stream);
  const bool fast_ok = (head_dim == 16 || head_dim == 32 || head_dim == 64 || head_dim == 128) &&
                       ldq % 4 == 0 && ((uintptr_t)sqkv & 15) == 0 &&
                       ((uintptr_t)kcache & 15) == 0 && ((uintptr_t)vcache & 15) == 0;
  if (fast_ok) {
    size_t smem = (size_t)wpb * (2 * max_len + 2) * 4;
#define FQ_SELF(KV, HD)                                                                      \
  launch_self_fast<KV, HD>(grid, smem, s, sqkv, ldq, kcache, vcache, hist, d_cur, rows, heads, \
                           max_len, scale, out, out16, ldo, exact)
    if (kv_dtype == FQ_F32) {
      if (head_dim == 16) FQ_SELF(float, 16);
      else if (head_dim == 32) FQ_SELF(float, 32);
      else if (head_dim == 64) FQ_SELF(float, 64);
      else FQ_SELF(float, 128);
    } else {
      if (head_dim == 16) FQ_SELF(h16, 16);
      else if (head_dim == 32) FQ_SELF(h16, 32);
      else if (head_dim == 64) FQ_SELF(h16, 64);
      else FQ_SELF(h16, 128);
    }
#undef FQ_SELF
    return launch_status("fq_decoder_self_attention");
  }
  size_t smem = (size_t)wpb * (max_len + 1) * 4;
  if (kv_dtype == FQ_F32) {
    launch_kernel(decoder_self_attention_kernel<float>, grid, wpb * 32, smem, s, 1u, 
        sqkv, ldq, (float*)kcache, (float*)vcache, hist, d_cur, (int)rows, (int)heads,
        (int)head_dim, (int)max_len, scale, out, reinterpret_cast<fq::h16*>(out16), ldo,
        exact);
  } else {
    launch_kernel(decoder_self_attention_kernel<h16>, grid, wpb * 32, smem, s, 1u, 
        sqkv, ldq, (h16*)kcache, (h16*)vcache, hist, d_cur, (int)rows,
        (int)heads, (int)head_dim, (int)max_len, scale, out,
        reinterpret_cast<fq::h16*>(out16), ldo, exact);
  }
  return launch_status("fq_decoder_self_attention");
}

int fq_decoder_self_attention_xh(const float* sqkv, int64_t ldq, void* kcache, void* vcache,
                                 int64_t plane, const int32_t* hist, const int32_t* d_cur,
                                 int64_t rows, int64_t heads, int64_t head_dim, int64_t max_len,
                                 float scale, float* out, void* out_hi, void* out_lo,
                                 int64_t ldo, fq_stream_t stream) {
  FQ_CHECK_ARG(sqkv && kcache && vcache && hist && d_cur && (out || out_hi) &&
                   (!out_hi == !out_lo) && rows > 0 && heads > 0 && max_len > 0 &&
                   (head_dim == 16 || head_dim == 32 || head_dim == 64 || head_dim == 128) &&
                   ldq % 2 == 0 && ((uintptr_t)sqkv & 7) == 0 && plane % 8 == 0 &&
                   ((uintptr_t)kcache & 15) == 0 && ((uintptr_t)vcache & 15) == 0,
               FQ_ERR_DIMENSION, "fq_decoder_self_attention_xh: bad args");
  FQ_CHECK_ARG(plane < (1LL << 31), FQ_ERR_CAPACITY, "fq_decoder_self_attention_xh: cache too large");
  const size_t smem = (size_t)(max_len + 16) * 4 + (size_t)max_len * 4;
  FQ_CHECK_ARG(smem <= 200 * 1024, FQ_ERR_CAPACITY, "decoder self-attention: max_len too long");
  const dim3 grid((unsigned)rows, (unsigned)heads);
  // ring depth: 2 (+1% over 3 at C2, measured; FQ_XH_SELF_STAGES=3 for A/B)
  static int ns = -1;
  if (ns < 0) {
    const char* e = getenv("FQ_XH_SELF_STAGES");
    ns = (e && e[0] == '3') ? 3 : 2;
  }
#define FQ_SELF_XH(HD)                                                                        \
  launch_kernel(ns == 3 ? decoder_self_attention_xh<HD, 3> : decoder_self_attention_xh<HD, 2>, \
                grid, 32, smem, as_stream(stream), 1u, sqkv,                                  \
                ldq, (h16*)kcache, (h16*)vcache, plane, hist, d_cur, (int)rows, (int)heads,    \
                (int)max_len, scale, out, (h16*)out_hi, (h16*)out_lo, ldo)
  if (head_dim == 16) FQ_SELF_XH(16);
  else if (head_dim == 32) FQ_SELF_XH(32);
  else if (head_dim == 64) FQ_SELF_XH(64);
  else FQ_SELF_XH(128);
#undef FQ_SELF_XH
  return launch_status("fq_decoder_self_attention_xh");
}

int fq_decoder_self_attention_xh_items(const float* sqkv, int64_t ldq, void* kcache,
                                       void* vcache, int64_t plane, const int32_t* hist,
                                       const int32_t* d_cur, int64_t items, int64_t beam,
                                       int64_t heads, int64_t head_dim, int64_t max_len,
                                       float scale, float* out, void* out_hi, void* out_lo,
                                       int64_t ldo, fq_stream_t stream) {
  FQ_CHECK_ARG(sqkv && kcache && vcache && hist && d_cur && (out || out_hi) &&
                   (!out_hi == !out_lo) && items > 0 && beam >= 1 && beam <= 8 && heads > 0 &&
                   max_len > 0 && head_dim == 64 && ldq % 2 == 0 && ((uintptr_t)sqkv & 7) == 0 &&
                   plane % 8 == 0 && ((uintptr_t)kcache & 15) == 0 &&
                   ((uintptr_t)vcache & 15) == 0,
               FQ_ERR_DIMENSION, "fq_decoder_self_attention_xh_items: bad args");
  FQ_CHECK_ARG(plane < (1LL << 31) && beam * max_len <= 32767, FQ_ERR_CAPACITY,
               "fq_decoder_self_attention_xh_items: cache too large");
  const int64_t dmax = beam * max_len, dpad = (dmax + 15) & ~15LL;
  static int ns = -1, nw = -1;  // ring depth / warps per CTA (FQ_XH_ITEMS_STAGES, _WARPS: A/B)
  if (ns < 0) {
    const char* e = getenv("FQ_XH_ITEMS_STAGES");
    ns = (e && e[0] == '2') ? 2 : 3;
    e = getenv("FQ_XH_ITEMS_WARPS");
    nw = e ? atoi(e) : 2;
    if (nw != 1 && nw != 4) nw = 2;
  }
  const size_t smem = (size_t)(dpad * beam + nw * (max_len + 16) + dmax) * 4 + (size_t)dmax * 2;
  FQ_CHECK_ARG(smem <= 160 * 1024, FQ_ERR_CAPACITY,
               "decoder self-attention (items): beam x max_len too large");
  const dim3 grid((unsigned)items, (unsigned)heads);
  auto kern = nw == 1   ? (ns == 3 ? self_attention_items_xh<1, 3> : self_attention_items_xh<1, 2>)
              : nw == 2 ? (ns == 3 ? self_attention_items_xh<2, 3> : self_attention_items_xh<2, 2>)
                        : self_attention_items_xh<4, 2>;  // (48 KB static smem cap)
  launch_kernel(kern, grid, 32 * nw, smem, as_stream(stream), 1u, sqkv, ldq, (h16*)kcache, (h16*)vcache, plane, hist,
                d_cur, (int)(items * beam), (int)beam, (int)heads, (int)max_len, scale, out,
                (h16*)out_hi, (h16*)out_lo, ldo);
  return launch_status("fq_decoder_self_attention_xh_items");
}

static int cross_xh_launch(const float* cq, int64_t ldcq, const void* ck, const void* cv,
                           int64_t plane, int64_t ldkv, int64_t batch, int64_t beam, int64_t seq,
                           int64_t heads, int64_t head_dim, float scale, const float* mask,
                           float* out, void* out_hi, void* out_lo, int64_t ldo, int* d_bad,
                           int nslab, int64_t qslab, const float* qbias, fq_stream_t stream) {
  FQ_CHECK_ARG(cq && ck && cv && (out || out_hi) && (!out_hi == !out_lo) && batch > 0 &&
                   beam > 0 && beam <= 8 && seq > 0 && seq <= 128 && heads > 0 &&
                   (head_dim == 16 || head_dim == 32 || head_dim == 64 || head_dim == 128) &&
                   ldcq % 2 == 0 && ((uintptr_t)cq & 7) == 0 && ldkv % 8 == 0 && plane % 8 == 0 &&
                   ((uintptr_t)ck & 15) == 0 && ((uintptr_t)cv & 15) == 0,
               FQ_ERR_DIMENSION, "fq_cross_attention_xh: unsupported shape");
  const dim3 grid((unsigned)batch, (unsigned)heads);
  const int nt = (int)((seq + 15) / 16);
  const size_t smem = 0;
  static int ns = -1;  // ring depth (FQ_XH_CROSS_STAGES = 2 | 3 | 4 | 6, A/B)
  if (ns < 0) {
    const char* e = getenv("FQ_XH_CROSS_STAGES");
    ns = e ? atoi(e) : 3;
    if (ns != 2 && ns != 4 && ns != 6) ns = 3;
  }
#define FQ_CROSS_XH(HD, NT)                                                                   \
  launch_kernel(ns == 2 ? cross_attention_xh<HD, NT, 2>                                       \
                : ns == 4 ? cross_attention_xh<HD, NT, 4>                                     \
                : ns == 6 ? cross_attention_xh<HD, NT, (HD <= 64 ? 6 : 3)>                    \
                          : cross_attention_xh<HD, NT, 3>,                                    \
                grid, 32, smem, as_stream(stream), 1u, cq, ldcq,                              \
                (const h16*)ck, (const h16*)cv, plane, ldkv, (int)beam, (int)seq, scale, mask, \
                out, (h16*)out_hi, (h16*)out_lo, ldo, d_bad, nslab, qslab, qbias)
#define FQ_CROSS_XHH(HD)                                                                      \
  if (nt == 1) FQ_CROSS_XH(HD, 1);                                                            \
  else if (nt == 2) FQ_CROSS_XH(HD, 2);                                                       \
  else if (nt == 3) FQ_CROSS_XH(HD, 3);                                                       \
  else if (nt == 4) FQ_CROSS_XH(HD, 4);                                                       \
  else FQ_CROSS_XH(HD, 8);
  if (head_dim == 16) { FQ_CROSS_XHH(16) }
  else if (head_dim == 32) { FQ_CROSS_XHH(32) }
  else if (head_dim == 64) { FQ_CROSS_XHH(64) }
  else { FQ_CROSS_XHH(128) }
#undef FQ_CROSS_XHH
#undef FQ_CROSS_XH
  return launch_status("fq_cross_attention_xh");
}

int fq_cross_attention_xh(const float* cq, int64_t ldcq, const void* ck, const void* cv,
                          int64_t plane, int64_t ldkv, int64_t batch, int64_t beam, int64_t seq,
                          int64_t heads, int64_t head_dim, float scale, const float* mask,
                          float* out, void* out_hi, void* out_lo, int64_t ldo, int* d_bad,
                          fq_stream_t stream) {
  return cross_xh_launch(cq, ldcq, ck, cv, plane, ldkv, batch, beam, seq, heads, head_dim, scale,
                         mask, out, out_hi, out_lo, ldo, d_bad, 0, 0, nullptr, stream);
}

int fq_cross_attention_xh_slabs(const float* q_slabs, int64_t nslab, int64_t ldq,
                                int64_t slab_stride, const float* q_bias, const void* ck,
                                const void* cv, int64_t plane, int64_t ldkv, int64_t batch,
                                int64_t beam, int64_t seq, int64_t heads, int64_t head_dim,
                                float scale, const float* mask, float* out, void* out_hi,
                                void* out_lo, int64_t ldo, int* d_bad, fq_stream_t stream) {
  FQ_CHECK_ARG(q_slabs && q_bias && nslab >= 1 && nslab <= 4 && slab_stride % 2 == 0 &&
                   ((uintptr_t)q_bias & 7) == 0,
               FQ_ERR_DIMENSION, "fq_cross_attention_xh_slabs: bad slabs");
  return cross_xh_launch(q_slabs, ldq, ck, cv, plane, ldkv, batch, beam, seq, heads, head_dim,
                         scale, mask, out, out_hi, out_lo, ldo, d_bad, (int)nslab, slab_stride,
                         q_bias, stream);
}

int fq_cross_attention_slabs(const float* q_slabs, int nslab, int64_t ldq, const float* q_bias,
                             const void* ck, const void* cv, int64_t ldkv, int64_t batch,
                             int64_t beam, int64_t seq, int64_t heads, int64_t head_dim,
                             float scale, const float* mask, float* out, void* out16, int64_t ldo,
                             int* d_bad, fq_stream_t stream) {
  FQ_CHECK_ARG(q_slabs && nslab >= 1 && nslab <= 8 && ck && cv && (out || out16) && batch > 0 &&
                   beam > 0 && beam <= 8 && seq > 0 && seq <= 64 && heads > 0 &&
                   head_dim == 64 && ldq % 2 == 0 && ((uintptr_t)q_slabs & 7) == 0 &&
                   ldkv % 8 == 0 && ((uintptr_t)ck & 15) == 0 && ((uintptr_t)cv & 15) == 0 &&
                   (!q_bias || ((uintptr_t)q_bias & 7) == 0),
               FQ_ERR_DIMENSION, "fq_cross_attention_slabs: unsupported shape");
  CUtensorMap tk, tv;
  const int64_t nrows = batch * seq, ncols = heads * head_dim;
  int rc;
  if ((rc = make_tmap_f16_sw128(&tk, ck, nrows, ncols, ldkv, 64, 64)) != FQ_OK) return rc;
  if ((rc = make_tmap_f16_sw128(&tv, cv, nrows, ncols, ldkv, 64, 64)) != FQ_OK) return rc;
  const int npairs = (int)(batch * heads);
  launch_kernel(cross_attention_tma, (unsigned)((npairs + kCrossWarps - 1) / kCrossWarps),
                32 * kCrossWarps, (size_t)kCrossWarps * 2 * 64 * 128 + 1024, as_stream(stream),
                1u, tk, tv, q_slabs, ldq, (int)beam, (int)seq, scale, mask, out,
                reinterpret_cast<fq::h16*>(out16), ldo, d_bad, (int)heads, npairs, nslab,
                (int64_t)(batch * beam) * ldq, q_bias);
  return launch_status("fq_cross_attention_slabs");
}

int fq_cross_attention(const float* cq, int64_t ldcq, const void* ck, const void* cv,
                       int kv_dtype, int64_t ldkv, int64_t batch, int64_t beam, int64_t seq,
                       int64_t heads, int64_t head_dim, float scale, const float* mask,
                       float* out, void* out16, int64_t ldo, int exact, int* d_bad,
                       fq_stream_t stream) {
  FQ_CHECK_ARG(cq && ck && cv && (out || out16) && batch > 0 && beam > 0 && seq > 0 &&
                   heads > 0 && head_dim > 0 && head_dim <= 128,
               FQ_ERR_DIMENSION, "fq_cross_attention: bad args");
  if (kv_dtype != FQ_F32 && !exact && head_dim == 64 && beam <= 8 && seq <= 64 &&
      ldcq % 2 == 0 && ((uintptr_t)cq & 7) == 0 && ldkv % 8 == 0 && ((uintptr_t)ck & 15) == 0 &&
      ((uintptr_t)cv & 15) == 0) {
    CUtensorMap tk, tv;
    const int64_t nrows = batch * seq, ncols = heads * head_dim;
    if (make_tmap_f16_sw128(&tk, ck, nrows, ncols, ldkv, 64, 64) == FQ_OK &&
        make_tmap_f16_sw128(&tv, cv, nrows, ncols, ldkv, 64, 64) == FQ_OK) {
      const int npairs = (int)(batch * heads);
      launch_kernel(cross_attention_tma, (unsigned)((npairs + kCrossWarps - 1) / kCrossWarps),
                    32 * kCrossWarps, (size_t)kCrossWarps * 2 * 64 * 128 + 1024,
                    as_stream(stream), 1u, tk, tv, cq, ldcq, (int)beam, (int)seq, scale, mask,
                    out, reinterpret_cast<fq::h16*>(out16), ldo, d_bad, (int)heads,
                    npairs, 0, (int64_t)0, (const float*)nullptr);
      return launch_status("fq_cross_attention");
    }
  }
  if (kv_dtype != FQ_F32 && !exact && (head_dim == 32 || head_dim == 64 || head_dim == 128) &&
      beam <= 8 && seq <= 64 && ldcq % 2 == 0 && ((uintptr_t)cq & 7) == 0 && ldkv % 8 == 0 &&
      ((uintptr_t)ck & 15) == 0 && ((uintptr_t)cv & 15) == 0) {
    const dim3 grid((unsigned)batch, (unsigned)heads);
    const int nt = (int)((seq + 15) / 16);
    const size_t msmem = (size_t)2 * nt * 16 * (head_dim * 2 + 16);
#define FQ_CROSS_M(HD, NT)                                                                     \
  launch_kernel(cross_attention_mma<HD, NT>, grid, 32, msmem, as_stream(stream), 1u, cq, ldcq,  \
                (const h16*)ck, (const h16*)cv, ldkv, (int)beam, (int)seq,  \
                scale, mask, out, reinterpret_cast<fq::h16*>(out16), ldo, d_bad)
#define FQ_CROSS_MH(HD)                      \
  if (nt == 1) FQ_CROSS_M(HD, 1);            \
  else if (nt == 2) FQ_CROSS_M(HD, 2);       \
  else if (nt == 3) FQ_CROSS_M(HD, 3);       \
  else FQ_CROSS_M(HD, 4);
    if (head_dim == 32) { FQ_CROSS_MH(32) }
    else if (head_dim == 64) { FQ_CROSS_MH(64) }
    else { FQ_CROSS_MH(128) }
#undef FQ_CROSS_MH
#undef FQ_CROSS_M
    return launch_status("fq_cross_attention");
  }
  dim3 grid((unsigned)(batch * heads));
  const size_t es = kv_dtype == FQ_F32 ? 4 : 2;
  const size_t fast_smem = (size_t)seq * (2 * head_dim + 16 / es) * es +
                           (size_t)beam * (head_dim + seq) * 4;
  const bool fast_ok = (head_dim == 64 || head_dim == 128 || head_dim == 32) &&
                       fast_smem <= 200 * 1024 && ldcq % 4 == 0 && ((uintptr_t)cq & 15) == 0 &&
                       (ldkv * es) % 16 == 0 && ((uintptr_t)ck & 15) == 0 &&
                       ((uintptr_t)cv & 15) == 0 && ldo % 2 == 0;
  if (fast_ok) {
    cudaStream_t s = as_stream(stream);
#define FQ_CROSS(KV, HD)                                                                   \
  launch_kernel(cross_attention_fast<KV, HD>, grid, 128, fast_smem, s, 1u,                                \
      cq, ldcq, (const KV*)ck, (const KV*)cv, ldkv, (int)beam, (int)seq, (int)heads, scale, \
      mask, out, reinterpret_cast<fq::h16*>(out16), ldo, exact, d_bad)
    if (kv_dtype == FQ_F32) {
      if (head_dim == 32) FQ_CROSS(float, 32);
      else if (head_dim == 64) FQ_CROSS(float, 64);
      else FQ_CROSS(float, 128);
    } else {
      if (head_dim == 32) FQ_CROSS(h16, 32);
      else if (head_dim == 64) FQ_CROSS(h16, 64);
      else FQ_CROSS(h16, 128);
    }
#undef FQ_CROSS
    return launch_status("fq_cross_attention");
  }
  const int threads = beam <= 4 ? 128 : 256;
  size_t smem = (size_t)(2 * seq * (head_dim + 1) + (threads / 32) * (seq + head_dim)) * 4;
  FQ_CHECK_ARG(smem <= 227 * 1024, FQ_ERR_CAPACITY, "cross attention: seq too long");
  if (kv_dtype == FQ_F32) {
    launch_kernel(cross_attention_kernel<float>, grid, threads, smem, as_stream(stream), 1u, 
        cq, ldcq, (const float*)ck, (const float*)cv, ldkv, (int)beam, (int)seq, (int)heads,
        (int)head_dim, scale, mask, out, reinterpret_cast<fq::h16*>(out16), ldo, exact,
        d_bad);
  } else {
    launch_kernel(cross_attention_kernel<h16>, grid, threads, smem, as_stream(stream), 1u, 
        cq, ldcq, (const h16*)ck, (const h16*)cv, ldkv, (int)beam,
        (int)seq, (int)heads, (int)head_dim, scale, mask, out,
        reinterpret_cast<fq::h16*>(out16), ldo, exact, d_bad);
  }
  return launch_status("fq_cross_attention");
}

}  // extern "C"
