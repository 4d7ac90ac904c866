// Device-resident top-k / top-p sampling step: the reference's
// Session._sampling_step (engine.py:175-195) over every row of one decode
// step, after the batched retrieve (decode.py:58-92) has left each live row's
// survivors x >= R (the row's true top-|C| tokens, |C| >= k).
//
// Per row (one CTA): the survivors sorted by (-logit, token) (_sorted_prefix,
// decode.py:389-396), the first k kept, probs = exp(f64(logit) - lse) in f64,
// and the inverse-CDF draw of _draw (decode.py:378-386): r = u * probs.sum()
// with numpy's pairwise summation order, c accumulated in order, the first
// token with r <= c (else the last). Top-p (k = 0): the whole sorted prefix,
// cut at the first cumulative sum >= p (np.searchsorted "left"), drawn the
// same way; a row whose survivors miss the nucleus mass (the reference would
// escalate its group count x8) sets err = 3 and the request re-runs on the
// host-driven path. The uniforms are the reference's own
// PCG64 stream, generated on the host in its order (one per live row per
// step, rows in batch order) and consumed here through a device draw counter:
// row b's draw is base + #{live rows before b}. The last CTA to finish
// advances the draw counter and the decode position (fq_step_advance).
#include "fq_common.cuh"

namespace fq {

constexpr int kSampThreads = 128;
constexpr int kSampCap = 1024;  // survivors ranked in shared memory; more -> error flag

// numpy's pairwise summation of a contiguous float64 array (np.add.reduce:
// blocks of 8 accumulators up to 128 elements, halves above; < 8 in order).
__device__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

__device__ __forceinline__ int block_count(int v, int* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// done: int32 [2][batch] (parity of the step: read [t & 1], write [(t+1) & 1]);
// out_tok int32 [batch][max_len]; out_len / fin int32 [batch]; dk_next int32
// [batch] (next step's retrieve group count: k live, 0 done); tokens int64
// [batch] (next step's input; 0 for done rows); draw int64 [1]; counters
// int32 [2] (arrival, live-after count); err int32 [1] (survivor overflow).
__global__ void __launch_bounds__(kSampThreads) sample_step_kernel(
    const float* __restrict__ logits, int64_t ld, const double* __restrict__ lse,
    const int32_t* __restrict__ cand_idx, int64_t cand_ld,
    const int64_t* __restrict__ cand_count, int k, double top_p, int groups, int V, int eos,
    const double* __restrict__ uniforms, int64_t n_uniforms, int64_t* draw, int32_t* done,
    int32_t* d_cur, int64_t max_steps, int max_len, int32_t* dk_next, int64_t* tokens,
    int32_t* out_tok, int32_t* out_len, int32_t* fin, int batch, int32_t* counters,
    int32_t* err) {
  pdl_enter();
  __shared__ int32_t s_tok[kSampCap];
  __shared__ float s_lg[kSampCap];
  __shared__ int32_t o_tok[kSampCap];
  __shared__ double o_p[kSampCap];
  __shared__ int red[kSampThreads / 32];
  __shared__ int s_last;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int t = *d_cur;
  const int32_t* done_in = done + (t & 1) * batch;
  int32_t* done_out = done + ((t + 1) & 1) * batch;
  const int64_t base = *draw;
  // live rows before b (the reference's draw order) and in total
  int before = 0, all = 0;
  for (int i = tid; i < batch; i += blockDim.x) {
    const int l = done_in[i] ? 0 : 1;
    all += l;
    before += i < b ? l : 0;
  }
  before = block_count(before, red);
  all = block_count(all, red);
  const bool live = !done_in[b];
  int d_out = 1;
  int32_t tok = 0;
  if (live) {
    const int64_t nc = cand_count[b];
    if (nc > kSampCap || nc < 1) {
      if (tid == 0) atomicExch(err, 1);
    } else {
      const int n = (int)nc;
      for (int j = tid; j < n; j += blockDim.x) {
        const int32_t tj = cand_idx[(int64_t)b * cand_ld + j];
        s_tok[j] = tj;
        s_lg[j] = logits[(int64_t)b * ld + tj];
      }
      __syncthreads();
      const int m = k > 0 ? min(k, n) : n;  // top-p: the whole sorted prefix
      for (int j = tid; j < n; j += blockDim.x) {  // rank under (-logit, token)
        const float v = s_lg[j];
        const int32_t tj = s_tok[j];
        int r = 0;
        for (int q = 0; q < n; ++q) {
          const float vq = s_lg[q];
          r += (vq > v || (vq == v && s_tok[q] < tj)) ? 1 : 0;
        }
        if (r < m) {
          o_tok[r] = tj;
          o_p[r] = exp((double)v - lse[b]);
        }
      }
      __syncthreads();
      if (tid == 0) {
        const int64_t ui = base + before;
        const double u = ui < n_uniforms ? uniforms[ui] : 0.0;
        if (ui >= n_uniforms) atomicExch(err, 2);
        int md = m;  // the draw's prefix length
        bool ok = true;
        if (k <= 0) {  // nucleus (decode.py:412-430): cut = searchsorted(cumsum, p, "left")
          double cs = 0.0;
          int cut = -1;
          for (int i = 0; i < n; ++i) {
            cs += o_p[i];
            if (cut < 0 && cs >= top_p) cut = i;
          }
          if (!(cs >= top_p || groups >= V)) {
            ok = false;  // the survivors miss the nucleus: the reference escalates x8
            atomicExch(err, 3);
          }
          md = min(cut < 0 ? n : cut, n - 1) + 1;
        }
        const double r = ok ? u * np_pairwise_sum(o_p, md) : 0.0;
        double c = 0.0;
        tok = o_tok[md - 1];
        for (int i = 0; i < md; ++i) {
          c += o_p[i];
          if (r <= c) {
            tok = o_tok[i];
            break;
          }
        }
        if (t < max_len) out_tok[(int64_t)b * max_len + t] = tok;
        out_len[b] = t + 1;
        if (tok == eos) fin[b] = 1;
        d_out = (tok == eos || (int64_t)t == max_steps - 1) ? 1 : 0;
      }
    }
  }
  if (tid == 0) {
    done_out[b] = d_out;
    dk_next[b] = d_out ? 0 : (k > 0 ? k : groups);
    tokens[b] = d_out ? 0 : tok;
    __threadfence();
    const int prev = atomicAdd(&counters[0], 1);
    s_last = prev == batch - 1;
  }
  __syncthreads();
  if (s_last) {  // every row has read d_cur / draw and written its flags
    __threadfence();
    int nl = 0;
    for (int i = tid; i < batch; i += blockDim.x) nl += __ldcg(done_out + i) ? 0 : 1;
    nl = block_count(nl, red);
    if (tid == 0) {
      counters[0] = 0;
      counters[1] = nl;
      *draw = base + all;
      *d_cur = t + 1;
    }
  }
}

}  // namespace fq

extern "C" int fq_sample_step(const float* logits, int64_t ld, const double* lse,
                              const int32_t* cand_idx, int64_t cand_ld, const int64_t* cand_count,
                              int64_t batch, int64_t k, double top_p, int64_t groups,
                              int64_t vocab, int64_t eos, const double* uniforms,
                              int64_t n_uniforms, int64_t* draw, int32_t* done, int32_t* d_cur,
                              int64_t max_steps, int64_t max_len, int32_t* dk_next,
                              int64_t* tokens, int32_t* out_tok, int32_t* out_len, int32_t* fin,
                              int32_t* counters, int32_t* err, fq_stream_t stream) {
  FQ_CHECK_ARG(logits && lse && cand_idx && cand_count && uniforms && draw && done && d_cur &&
                   dk_next && tokens && out_tok && out_len && fin && counters && err &&
                   batch > 0 && ld >= 1 && cand_ld >= 1 && max_len >= 1,
               FQ_ERR_DIMENSION, "fq_sample_step: bad args");
  FQ_CHECK_ARG((k >= 1 && k <= fq::kSampCap) || (k == 0 && top_p > 0.0 && top_p <= 1.0),
               FQ_ERR_PARAMETER, "fq_sample_step: k outside [1, 1024] / p outside (0, 1]");
  fq::launch_kernel(fq::sample_step_kernel, (unsigned)batch, fq::kSampThreads, 0,
                fq::as_stream(stream), 1u, logits, ld, lse, cand_idx, cand_ld, cand_count, (int)k,
                top_p, (int)groups, (int)vocab, (int)eos, uniforms, n_uniforms, draw, done, d_cur, max_steps, (int)max_len,
                dk_next, tokens, out_tok, out_len, fin, (int)batch, counters, err);
  return fq::launch_status("fq_sample_step");
}
