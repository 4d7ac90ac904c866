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
// 128-bit loads (8 bf16 or 4 fp32 per load), all issued before first use.
#include "fq_common.cuh"

namespace fq {

template <typename T>
__device__ __forceinline__ float ld_as_f32(const T* p);
template <>
__device__ __forceinline__ float ld_as_f32<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_as_f32<__nv_bfloat16>(const __nv_bfloat16* p) {
  return bf2f(*p);
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
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& raw, float* o) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = __uint_as_float(w[i] << 16);
    o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
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
                                            __nv_bfloat16* out16, int* d_bad) {
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
    if (out16) out16[e] = f2bf(acc);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Encoder self-attention: CTA per (item, head); K/V of the head in smem.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) encoder_attention_kernel(
    const float* __restrict__ qkv, int64_t ldq, int seq, int heads, int hd, float scale,
    const float* __restrict__ mask, float* __restrict__ out, __nv_bfloat16* __restrict__ out16,
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
    int max_len, float scale, float* __restrict__ out, __nv_bfloat16* __restrict__ out16,
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
      kc[slot_cur + e] = f2bf(rowp[d + e]);
      vc[slot_cur + e] = f2bf(rowp[2 * d + e]);
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
          if constexpr (sizeof(KV) == 2) kv = bf2f(f2bf(kv));  // the stored (rounded) key
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
      if (out16) out16[o + e] = f2bf(acc[i]);
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
    const float* __restrict__ mask, float* __restrict__ out, __nv_bfloat16* __restrict__ out16,
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
// softmax, and P.V with paired columns (bf16x2 / float2 loads).
template <typename KV, int HD>
__global__ void __launch_bounds__(128) cross_attention_fast(
    const float* __restrict__ cq, int64_t ldcq, const KV* __restrict__ ck,
    const KV* __restrict__ cv, int64_t ldkv, int beam, int seq, int heads, float scale,
    const float* __restrict__ mask, float* __restrict__ out, __nv_bfloat16* __restrict__ out16,
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
        v0 = __uint_as_float(raw << 16);
        v1 = __uint_as_float(raw & 0xffff0000u);
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
    if (out16) *reinterpret_cast<__nv_bfloat162*>(out16 + o) = __floats2bfloat162_rn(a0, a1);
  }
}

// Generic decoder self-attention (any head_dim <= 128), warp-reduced dots.
template <typename KV>
__global__ void __launch_bounds__(128) decoder_self_attention_kernel(
    const float* __restrict__ sqkv, int64_t ldq, KV* __restrict__ kc, KV* __restrict__ vc,
    const int32_t* __restrict__ hist, const int32_t* __restrict__ d_cur, int rows, int heads,
    int hd, int max_len, float scale, float* __restrict__ out,
    __nv_bfloat16* __restrict__ out16, int64_t ldo, int exact) {
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
        kc[slot_cur + e] = f2bf(kn[i]);
        vc[slot_cur + e] = f2bf(vn[i]);
        kn[i] = bf2f(f2bf(kn[i]));
        vn[i] = bf2f(f2bf(vn[i]));
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
      if (out16) out16[o + e] = f2bf(acc[i]);
    }
  }
}

int attention_prepare() {
  const int big = 227 * 1024;
  if (cudaFuncSetAttribute(encoder_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_kernel<__nv_bfloat16>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_fast<float, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<float, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<float, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<__nv_bfloat16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<__nv_bfloat16, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
      cudaFuncSetAttribute(cross_attention_fast<__nv_bfloat16, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) {
    set_error("fq_prepare: cannot opt in to large shared memory (attention)");
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

template <typename KV, int HD>
static void launch_self_fast(dim3 grid, size_t smem, cudaStream_t s, const float* sqkv,
                             int64_t ldq, void* kc, void* vc, const int32_t* hist,
                             const int32_t* d_cur, int64_t rows, int64_t heads, int64_t max_len,
                             float scale, float* out, void* out16, int64_t ldo, int exact) {
  launch_kernel(decoder_self_attention_fast<KV, HD>, grid, 128, smem, s, 1u, 
      sqkv, ldq, (KV*)kc, (KV*)vc, hist, d_cur, (int)rows, (int)heads, (int)max_len, scale, out,
      reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact);
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
  const int threads = 256;
  size_t smem = (size_t)(2 * seq * (head_dim + 1) + seq * head_dim + (threads / 32) * seq) * 4;
  FQ_CHECK_ARG(smem <= 227 * 1024, FQ_ERR_CAPACITY, "encoder attention: seq %lld too long",
               (long long)seq);
  launch_kernel(encoder_attention_kernel, (unsigned)(batch * heads), threads, smem, as_stream(stream), 1u, 
      qkv, ldq, (int)seq, (int)heads, (int)head_dim, scale, mask, out,
      reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact, d_bad);
  return launch_status("fq_encoder_attention");
}

int fq_decoder_self_attention(const float* sqkv, int64_t ldq, void* kcache, void* vcache,
                              int kv_dtype, const int32_t* hist, const int32_t* d_cur,
                              int64_t rows, int64_t heads, int64_t head_dim, int64_t max_len,
                              float scale, float* out, void* out16, int64_t ldo, int exact,
                              fq_stream_t stream) {
  FQ_CHECK_ARG(sqkv && kcache && vcache && hist && d_cur && (out || out16) && rows > 0 &&
                   heads > 0 && head_dim > 0 && head_dim <= 128 && max_len > 0,
               FQ_ERR_DIMENSION, "fq_decoder_self_attention: bad args");
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
      if (head_dim == 16) FQ_SELF(__nv_bfloat16, 16);
      else if (head_dim == 32) FQ_SELF(__nv_bfloat16, 32);
      else if (head_dim == 64) FQ_SELF(__nv_bfloat16, 64);
      else FQ_SELF(__nv_bfloat16, 128);
    }
#undef FQ_SELF
    return launch_status("fq_decoder_self_attention");
  }
  size_t smem = (size_t)wpb * (max_len + 1) * 4;
  if (kv_dtype == FQ_F32) {
    launch_kernel(decoder_self_attention_kernel<float>, grid, wpb * 32, smem, s, 1u, 
        sqkv, ldq, (float*)kcache, (float*)vcache, hist, d_cur, (int)rows, (int)heads,
        (int)head_dim, (int)max_len, scale, out, reinterpret_cast<__nv_bfloat16*>(out16), ldo,
        exact);
  } else {
    launch_kernel(decoder_self_attention_kernel<__nv_bfloat16>, grid, wpb * 32, smem, s, 1u, 
        sqkv, ldq, (__nv_bfloat16*)kcache, (__nv_bfloat16*)vcache, hist, d_cur, (int)rows,
        (int)heads, (int)head_dim, (int)max_len, scale, out,
        reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact);
  }
  return launch_status("fq_decoder_self_attention");
}

int fq_cross_attention(const float* cq, int64_t ldcq, const void* ck, const void* cv,
                       int kv_dtype, int64_t ldkv, int64_t batch, int64_t beam, int64_t seq,
                       int64_t heads, int64_t head_dim, float scale, const float* mask,
                       float* out, void* out16, int64_t ldo, int exact, int* d_bad,
                       fq_stream_t stream) {
  FQ_CHECK_ARG(cq && ck && cv && (out || out16) && batch > 0 && beam > 0 && seq > 0 &&
                   heads > 0 && head_dim > 0 && head_dim <= 128,
               FQ_ERR_DIMENSION, "fq_cross_attention: bad args");
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
      mask, out, reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact, d_bad)
    if (kv_dtype == FQ_F32) {
      if (head_dim == 32) FQ_CROSS(float, 32);
      else if (head_dim == 64) FQ_CROSS(float, 64);
      else FQ_CROSS(float, 128);
    } else {
      if (head_dim == 32) FQ_CROSS(__nv_bfloat16, 32);
      else if (head_dim == 64) FQ_CROSS(__nv_bfloat16, 64);
      else FQ_CROSS(__nv_bfloat16, 128);
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
        (int)head_dim, scale, mask, out, reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact,
        d_bad);
  } else {
    launch_kernel(cross_attention_kernel<__nv_bfloat16>, grid, threads, smem, as_stream(stream), 1u, 
        cq, ldcq, (const __nv_bfloat16*)ck, (const __nv_bfloat16*)cv, ldkv, (int)beam,
        (int)seq, (int)heads, (int)head_dim, scale, mask, out,
        reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact, d_bad);
  }
  return launch_status("fq_cross_attention");
}

}  // extern "C"
