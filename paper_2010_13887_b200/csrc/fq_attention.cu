// Fused attention for the device engine.
//
// The reference runs attention as gemm_batched(QK^T) -> scale_mask_softmax ->
// gemm_batched(P.V) writing a merged-head strided view (model.py:329-336,
// :572-580, :597-604). These kernels do the same three steps in one pass per
// (item, head) so the [b, h, q, l] score tensor never reaches HBM; the softmax
// keeps the kernels.py:106-139 numerics in exact mode (fp32 scale+mask, f64
// exp and sum, F32(exp * (1/sum)), masked -> 0). Every dot product is an fp32
// FMA chain; the P.V sum runs over keys in ascending order.
//
// Decoder self-attention replaces the reference's ping-pong KV gather
// (kernels.py:189-201: ~50 GB/request at C2) with a copy-free
// history table: slot (t, r) of the cache is written once, by row r at step t,
// and hist[r, t] names the physical row whose slot holds row r's position t.
// Beam reorder then moves B*K*max_len int32 instead of the K/V history.
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

// ---------------------------------------------------------------------------
// Encoder self-attention: CTA per (item, head); K/V of the head in smem.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) encoder_attention_kernel(
    const float* __restrict__ qkv, int64_t ldq, int seq, int heads, int hd, float scale,
    const float* __restrict__ mask, float* __restrict__ out, __nv_bfloat16* __restrict__ out16,
    int64_t ldo, int exact, int* d_bad) {
  extern __shared__ float sm[];
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int d = heads * hd;
  const int hp = hd + 1;  // padded row: conflict-free column walks
  float* Ks = sm;
  float* Vs = Ks + seq * hp;
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Ss = Vs + seq * hp + w * (seq + hd);  // per-warp scores
  float* Qs = Ss + seq;                        // per-warp query
  const float* base = qkv + (int64_t)b * seq * ldq;
  for (int i = threadIdx.x; i < seq * hd; i += blockDim.x) {
    int s = i / hd, e = i % hd;
    Ks[s * hp + e] = base[s * ldq + d + h * hd + e];
    Vs[s * hp + e] = base[s * ldq + 2 * d + h * hd + e];
  }
  __syncthreads();
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  for (int i = w; i < seq; i += nw) {
    for (int e = lane; e < hd; e += 32) Qs[e] = base[i * ldq + h * hd + e];
    __syncwarp();
    for (int j = lane; j < seq; j += 32) {
      float acc = 0.0f;
      for (int e = 0; e < hd; ++e) acc = fmaf(Qs[e], Ks[j * hp + e], acc);
      float t = fmul_rn(acc, scale);
      if (mk) t = fadd_rn(t, mk[j]);
      Ss[j] = t;
    }
    __syncwarp();
    bool ok = warp_softmax(Ss, seq, exact);
    if (!ok) {
      if (lane == 0 && d_bad) atomicAdd(d_bad, 1);
      continue;
    }
    const int64_t orow = ((int64_t)b * seq + i) * ldo + h * hd;
    for (int e = lane; e < hd; e += 32) {
      float acc = 0.0f;
      for (int j = 0; j < seq; ++j) acc = fmaf(Ss[j], Vs[j * hp + e], acc);
      if (out) out[orow + e] = acc;
      if (out16) out16[orow + e] = f2bf(acc);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Decoder self-attention, warp per (row, head); 4 consecutive rows (one item
// at beam 4) share a CTA so beams reading the same physical slots hit L1.
// ---------------------------------------------------------------------------
template <typename KV>
__global__ void __launch_bounds__(128) decoder_self_attention_kernel(
    const float* __restrict__ sqkv, int64_t ldq, KV* __restrict__ kc, KV* __restrict__ vc,
    const int32_t* __restrict__ hist, const int32_t* __restrict__ d_cur, int rows, int heads,
    int hd, int max_len, float scale, float* __restrict__ out,
    __nv_bfloat16* __restrict__ out16, int64_t ldo, int exact) {
  extern __shared__ float sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + w;
  const int h = blockIdx.y;
  if (r >= rows) return;
  const int cur = *d_cur;
  const int d = heads * hd;
  float* Ss = sm + w * (max_len + 1);
  const float* row = sqkv + (int64_t)r * ldq;
  // this step's K/V: used for position cur and stored into slot (cur, r)
  const int64_t slot_cur = ((int64_t)cur * rows + r) * d + h * hd;
  constexpr int EPL = 4;  // head_dim <= 128: up to 4 elements per lane
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
        kn[i] = bf2f(f2bf(kn[i]));  // attend to the stored (rounded) value
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
  warp_softmax(Ss, cur + 1, exact);  // no mask: causality is implicit (model.py:576)
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
  extern __shared__ float sm[];
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int hp = hd + 1;
  float* Ks = sm;
  float* Vs = Ks + seq * hp;
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Ss = Vs + seq * hp + w * (seq + hd);
  float* Qs = Ss + seq;
  for (int i = threadIdx.x; i < seq * hd; i += blockDim.x) {
    int s = i / hd, e = i % hd;
    int64_t src = ((int64_t)b * seq + s) * ldkv + h * hd + e;
    Ks[s * hp + e] = ld_as_f32(ck + src);
    Vs[s * hp + e] = ld_as_f32(cv + src);
  }
  __syncthreads();
  const float* mk = mask ? mask + (int64_t)b * seq : nullptr;
  for (int i = w; i < beam; i += nw) {
    const int64_t r = (int64_t)b * beam + i;
    for (int e = lane; e < hd; e += 32) Qs[e] = cq[r * ldcq + h * hd + e];
    __syncwarp();
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
      continue;
    }
    for (int e = lane; e < hd; e += 32) {
      float acc = 0.0f;
      for (int j = 0; j < seq; ++j) acc = fmaf(Ss[j], Vs[j * hp + e], acc);
      if (out) out[r * ldo + h * hd + e] = acc;
      if (out16) out16[r * ldo + h * hd + e] = f2bf(acc);
    }
    __syncwarp();
  }
}

int attention_prepare() {
  const int big = 227 * 1024;
  if (cudaFuncSetAttribute(encoder_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) ||
      cudaFuncSetAttribute(cross_attention_kernel<__nv_bfloat16>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, big)) {
    set_error("fq_prepare: cannot opt in to large shared memory (attention)");
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
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
  size_t smem = (size_t)(2 * seq * (head_dim + 1) + (threads / 32) * (seq + head_dim)) * 4;
  FQ_CHECK_ARG(smem <= 227 * 1024, FQ_ERR_CAPACITY, "encoder attention: seq %lld too long",
               (long long)seq);
  encoder_attention_kernel<<<(unsigned)(batch * heads), threads, smem, as_stream(stream)>>>(
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
  size_t smem = (size_t)wpb * (max_len + 1) * 4;
  if (kv_dtype == FQ_F32) {
    decoder_self_attention_kernel<float><<<grid, wpb * 32, smem, as_stream(stream)>>>(
        sqkv, ldq, (float*)kcache, (float*)vcache, hist, d_cur, (int)rows, (int)heads,
        (int)head_dim, (int)max_len, scale, out, reinterpret_cast<__nv_bfloat16*>(out16), ldo,
        exact);
  } else {
    decoder_self_attention_kernel<__nv_bfloat16><<<grid, wpb * 32, smem, as_stream(stream)>>>(
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
  const int threads = beam <= 4 ? 128 : 256;
  size_t smem = (size_t)(2 * seq * (head_dim + 1) + (threads / 32) * (seq + head_dim)) * 4;
  FQ_CHECK_ARG(smem <= 227 * 1024, FQ_ERR_CAPACITY, "cross attention: seq too long");
  dim3 grid((unsigned)(batch * heads));
  if (kv_dtype == FQ_F32) {
    cross_attention_kernel<float><<<grid, threads, smem, as_stream(stream)>>>(
        cq, ldcq, (const float*)ck, (const float*)cv, ldkv, (int)beam, (int)seq, (int)heads,
        (int)head_dim, scale, mask, out, reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact,
        d_bad);
  } else {
    cross_attention_kernel<__nv_bfloat16><<<grid, threads, smem, as_stream(stream)>>>(
        cq, ldcq, (const __nv_bfloat16*)ck, (const __nv_bfloat16*)cv, ldkv, (int)beam,
        (int)seq, (int)heads, (int)head_dim, scale, mask, out,
        reinterpret_cast<__nv_bfloat16*>(out16), ldo, exact, d_bad);
  }
  return launch_status("fq_cross_attention");
}

}  // extern "C"
